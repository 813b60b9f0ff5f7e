#!/bin/bash
# Interleaved A/B of library builds at 100^3 and 300^3: tools/gpu_ab3.sh OUT libA.so libB.so ...
D=gpurun_out/$1; shift; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for rep in 1 2 3; do for M in "100 100 100" "300 300 300"; do for L in "$@"; do
  MINIFE_LIB_PATH=$L timeout 300 python tools/ab_solve.py $M 4 >> $D/ab.jsonl 2>>$D/err.log
done; done; done
