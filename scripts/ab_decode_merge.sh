#!/bin/bash
# A/B of the decode kernel: library variants x separate / in-kernel merge
for k in "$@"; do
  for sep in ${SEPS:-1 0}; do
    PI_BENCH_SEPARATE_MERGE=$sep PACKINFER_LIB=$PWD/variants/libpi_$k.so timeout 300 python bench.py --no-e2e --no-cpu --no-mixed --no-loop --no-context --steps 30 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('$k sep=$sep','prefill',round(d['roofline']['kernel_ms'],3),'ms | cfg3 decode',round(d['decode']['kernel_ms'],3),'ms',round(d['decode']['achieved_gbs']),'GB/s | cfg4 decode',round(d['shared_prefix']['decode']['kernel_ms'],4),'ms',round(d['shared_prefix']['decode']['achieved_gbs']),'GB/s')"
  done
done
