#!/bin/bash
# A/B of the prefill LPT bucket width (plan.cpp PI_LPT_BUCKET_SHIFT): kernel time (cfg2, cfg5
# mixed fused) + DRAM bytes of the cfg2 prefill kernel.
for k in ${@:-0 3 5}; do
  PACKINFER_LIB=$PWD/variants/libpi_lpt$k.so timeout 300 python bench.py --no-e2e --no-cpu --no-decode --steps 20 2>/dev/null | tail -1 | python -c "import json,sys;d=json.load(sys.stdin);print('shift',$k,round(d['roofline']['achieved'],1),'TF/s',round(d['roofline']['kernel_ms'],3),'ms | cfg5 fused',round(d['mixed']['fused_attention_ms'],1),'ms',round(d['mixed']['tflops_fused'],1))"
  PACKINFER_LIB=$PWD/variants/libpi_lpt$k.so timeout 300 ncu --metrics dram__bytes_read.sum --clock-control none -k regex:packed_attention -c 3 --csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-decode --no-mixed 2>/dev/null | grep -E "dram__bytes" | tail -1 | awk -F, '{print "   dram read", $NF}'
done
