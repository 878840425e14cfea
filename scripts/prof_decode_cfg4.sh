#!/bin/bash
# ncu --set full of one configs[3] decode attention launch (+ SASS source page with stall samples)
OUT=gpurun_out/prof_${1:-cfg4}
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:packed_attention -s 2 -c 1 \
  -o $OUT/decode4 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-mixed --no-loop --no-decode > $OUT/decode4.log 2>&1
ncu -i $OUT/decode4.ncu-rep --page raw --csv > $OUT/decode4_raw.csv 2>/dev/null
ncu -i $OUT/decode4.ncu-rep --page source --csv --print-source sass > $OUT/decode4_sass.csv 2>/dev/null
python scripts/sass_hot.py $OUT/decode4_sass.csv 45 > $OUT/decode4_hot.txt 2>&1
head -3 $OUT/decode4_raw.csv | cut -c1-300
