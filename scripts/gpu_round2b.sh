#!/bin/bash
O=gpurun_out/r2b; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc $?"
tail -15 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc $?"
tail -3 $O/bench.err
