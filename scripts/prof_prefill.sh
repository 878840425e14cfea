#!/bin/bash
# One ncu --set full capture of the prefill attention kernel (+ SASS-level source page).
TAG=${1:-x}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:packed_attention -s 1 -c 1 \
  -o $OUT/prefill python bench.py --steps 1 --warmup 1 --no-decode --no-e2e --no-cpu > $OUT/prefill.log 2>&1
ncu -i $OUT/prefill.ncu-rep --page raw --csv > $OUT/prefill_raw.csv 2>/dev/null
ncu -i $OUT/prefill.ncu-rep --page source --csv --print-source sass > $OUT/prefill_sass.csv 2>/dev/null
ls -la $OUT
