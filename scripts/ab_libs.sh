#!/bin/bash
# A/B of library variants (variants/libpi_<name>.so) on the bench's prefill / decode kernels.
# Build a variant: python -c "from paper_2602_06072_b200 import build as B; B.build(True, False, 'variants/libpi_<name>.so', ('PI_SOME_FLAG=1',))"
for k in "$@"; do
  PACKINFER_LIB=$PWD/variants/libpi_$k.so timeout 300 python bench.py --no-e2e --no-cpu --no-mixed --no-loop --no-prefix --no-context --steps 30 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('$k',round(d['roofline']['achieved'],1),'TF/s',round(d['roofline']['kernel_ms'],3),'ms | decode',round(d['decode']['achieved_gbs']),'GB/s',round(d['decode']['kernel_ms'],3),'ms')"
done
