#!/bin/bash
# Interleaved A/B of ctx options: tools/gpu_opt_ab.sh OUT "NX NY NZ" "opt=a" "opt=b" ...
D=gpurun_out/$1; MESH=$2; shift 2; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for rep in 1 2 3; do for O in "$@"; do
  timeout 300 python tools/ab_solve.py $MESH 4 --opt $O >> $D/ab.jsonl 2>>$D/err.log
done; done
