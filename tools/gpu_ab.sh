#!/bin/bash
# Interleaved A/B of library builds: tools/gpu_ab.sh OUT "NX NY NZ" libA.so libB.so ...
D=gpurun_out/$1; MESH=$2; shift 2; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for rep in 1 2 3; do
  for L in "$@"; do
    MINIFE_LIB_PATH=$L timeout 300 python tools/ab_solve.py $MESH 5 >> $D/ab.jsonl 2>>$D/err.log
  done
done
