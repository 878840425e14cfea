#!/bin/bash
# Launch list + full ncu captures of the prefill / decode attention and relayout kernels
# (run under gpurun, 1 GPU).  Usage: scripts/profile.sh <tag>
set -u
TAG=${1:-r02}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-mixed --no-loop --no-prefix --no-context"
# launch list of one short bench (kernel durations, cold-cache + serialised: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches.csv $B > $OUT/launches_bench.log 2>&1
# prefill: the 2nd attention launch of the headline (timed step); decode: the 2nd of the cfg3 section
# (attention launches before it: headline warm-up + step = 2, sequential-latency runner 2 + 10 = 12,
# cfg3 warm-up 1 -> skip 15)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:packed_attention -s 1 -c 1 \
  -o $OUT/prefill $B --no-decode > $OUT/prefill.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:packed_attention -s 15 -c 1 \
  -o $OUT/decode $B > $OUT/decode.log 2>&1
# configs[3] decode: the 4th attention launch of the in-process harness (current library as variants/libpi_cur.so)
cp paper_2602_06072_b200/libpackinfer.so variants/libpi_cur.so
timeout 900 ncu --set full --clock-control none --import-source on -k regex:packed_attention -s 3 -c 1 \
  -o $OUT/decode_cfg4 python scripts/ab_inproc.py cfg4_decode cur --reps 2 > $OUT/decode_cfg4.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:relayout -s 1 -c 1 \
  -o $OUT/relayout $B --no-decode > $OUT/relayout.log 2>&1
for k in prefill decode decode_cfg4 relayout; do
  ncu -i $OUT/$k.ncu-rep --page raw --csv > $OUT/${k}_raw.csv 2>/dev/null
done
ncu -i $OUT/prefill.ncu-rep --page source --csv --print-source sass > $OUT/prefill_sass.csv 2>/dev/null
ls -la $OUT
