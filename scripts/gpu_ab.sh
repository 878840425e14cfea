#!/bin/bash
# usage: scripts/gpu_ab.sh <outdir> <test-variant or -> <variant>...  : optional GPU parity suite of one
# variant, then the prefill/decode kernel A/B of all variants, alternated twice
O=$1; shift; T=$1; shift; mkdir -p $O
if [ "$T" != "-" ]; then
  PACKINFER_LIB=$PWD/variants/libpi_$T.so timeout 600 python -m pytest tests -m gpu -x -q > $O/gpu_tests_$T.txt 2>&1
  tail -2 $O/gpu_tests_$T.txt
fi
for i in 1 2; do bash scripts/ab_libs.sh "$@"; done > $O/ab.txt 2>&1
cat $O/ab.txt
