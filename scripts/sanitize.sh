#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over small runs of every kernel:
# relayout, fused + split attention (prefill pair units, decode single units, splits + merge),
# fp32 toy path (kind::tf32 + V^T staging), decode group sharding.  Run under gpurun, 1 GPU.
set -u
OUT=gpurun_out/sanitizer_${1:-r02}
mkdir -p $OUT
PY="python scripts/dbg_sanitize.py"
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 $PY > $OUT/$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/summary.txt
done
cat $OUT/summary.txt
