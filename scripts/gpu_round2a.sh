#!/bin/bash
# GPU session: suite, bench, A/B of the P row-sum variants, 2-rank one-GPU self-launch smoke
O=gpurun_out/r2a; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "tests rc $?"
tail -3 $O/gpu_tests.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc $?"
tail -2 $O/bench.err
bash scripts/ab_libs.sh prod exactsum prod exactsum > $O/ab_rowsum.txt 2>&1; cat $O/ab_rowsum.txt
timeout 600 python scripts/ab_pv_precision.py > $O/ab_precision.txt 2>&1; cat $O/ab_precision.txt | cut -c1-300
PI_BENCH_ONE_GPU=1 timeout 600 python bench.py --gpus 2 --steps 10 --no-e2e --no-mixed --no-loop > $O/bench_2rank_onegpu.json 2> $O/bench_2rank.err; echo "2rank rc $?"
tail -3 $O/bench_2rank.err
