#!/bin/bash
# Interleaved A/B of prebuilt library variants (no tests): tools/gpu_ab_only.sh OUT "N1 N2" libA libB ...
D=gpurun_out/$1; SIZES=$2; shift 2; mkdir -p $D
for rep in 1 2; do for N in $SIZES; do for L in "$@"; do
  MINIFE_LIB_PATH=paper_1505_08023_b200/lib/alt_$L.so timeout 300 python tools/ab_solve.py $N $N $N 3 >> $D/ab.jsonl 2>>$D/err.log
done; done; done
