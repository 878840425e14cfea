#!/bin/bash
O=gpurun_out/r2c; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "tests rc $?"
tail -8 $O/gpu_tests.log
bash scripts/ab_libs.sh rs2 rs0 rs1 rs2 rs0 rs1 > $O/ab_rowsum.txt 2>&1; cat $O/ab_rowsum.txt
timeout 900 python scripts/ab_pv_precision.py > $O/ab_precision.txt 2>&1; cut -c1-200 $O/ab_precision.txt
timeout 300 python scripts/trace_decode.py cfg4_decode > $O/trace_cfg4.txt 2>&1; head -40 $O/trace_cfg4.txt
