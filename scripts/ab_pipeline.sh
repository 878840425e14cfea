#!/bin/bash
# A/B: headline steps pipelined (plan upload + relayout of step i+1 under attention i) vs sequential
for pl in 1 0 1 0 1 0; do
  PI_BENCH_PIPELINE=$pl timeout 300 python bench.py --no-e2e --no-cpu --no-mixed --no-loop --no-prefix --no-decode --no-context --steps 50 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('pipeline=$pl step',round(d['ms_per_step'],4),'kernel',round(d['roofline']['kernel_ms'],4),'value',round(d['value'],1))"
done
