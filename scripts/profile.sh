#!/bin/bash
# Launch list + one full ncu capture of the top kernel (run under gpurun, 1 GPU).
# Usage: scripts/profile.sh <tag>
set -u
TAG=${1:-r01}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
# every launch with device time (cold-cache, serialised: compare SHARES, not absolutes)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > $OUT/launches_bench.log 2>&1
# full capture of the prefill attention kernel (first launch after warm-up)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:packed_attention -s 1 -c 1 \
  -o $OUT/prefill python bench.py --steps 1 --warmup 1 --no-decode --no-e2e --no-cpu > $OUT/prefill.log 2>&1
# full capture of the decode attention kernel (cfg3): skip the prefill launches (2) and the first decode
timeout 900 ncu --set full --clock-control none --import-source on -k regex:packed_attention -s 3 -c 1 \
  -o $OUT/decode python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $OUT/decode.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:relayout -s 1 -c 1 \
  -o $OUT/relayout python bench.py --steps 1 --warmup 1 --no-decode --no-e2e --no-cpu > $OUT/relayout.log 2>&1
ls -la $OUT
