#!/bin/bash
# Interleaved A/B of ctx options at several sizes: tools/gpu_opts.sh OUT "N1 N2" "opt=a" "opt=b" ...
D=gpurun_out/$1; SIZES=$2; shift 2; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for rep in 1 2; do for N in $SIZES; do for O in "$@"; do
  timeout 300 python tools/ab_solve.py $N $N $N 3 --opt $O >> $D/ab.jsonl 2>>$D/err.log
done; done; done
