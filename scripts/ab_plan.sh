#!/bin/bash
# A/B of planner options on the bench's decode kernels: "flags:chunk" pairs, e.g. 0:1024 2:1024 0:2048
for fc in "$@"; do
  f=${fc%%:*}; c=${fc##*:}
  PI_BENCH_PLAN_FLAGS=$f PI_BENCH_DECODE_CHUNK=$c timeout 300 python bench.py --no-e2e --no-cpu --no-mixed --no-loop --no-context --steps 30 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);s=d['shared_prefix']['decode'];print('flags=$f chunk=$c | cfg3 decode',round(d['decode']['kernel_ms'],3),'ms',round(d['decode']['achieved_gbs']),'GB/s items',d['decode']['work_items'],'| cfg4 decode',round(s['kernel_ms'],4),'ms',round(s['achieved_gbs']),'GB/s items',s['work_items'])"
done
