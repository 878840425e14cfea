#!/bin/bash
# A/B of PI_POLY_PAIRS (exp2 pairs per 8 on the FMA pipe instead of MUFU): prefill + decode kernel time.
for k in ${@:-2 3}; do
  PACKINFER_LIB=$PWD/variants/libpi_poly$k.so timeout 300 python bench.py --no-e2e --no-cpu --no-mixed --no-loop --steps 20 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('poly',$k,round(d['roofline']['achieved'],1),'TF/s',round(d['roofline']['kernel_ms'],3),'ms | decode',round(d['decode']['achieved_gbs']),'GB/s',round(d['decode']['kernel_ms'],3),'ms')"
done
