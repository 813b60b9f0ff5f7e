#!/bin/bash
# A/B of library builds with a parity gate: tools/gpu_ab_parity.sh OUT libA.so libB.so ...
D=gpurun_out/$1; shift; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for L in "$@"; do
  MINIFE_LIB_PATH=$L timeout 600 python -m pytest tests/test_gpu_golden.py -m gpu -q -x -k "300cubed_bench or 400cubed_single" > $D/parity_$(basename $L).log 2>&1; echo "rc=$?" >> $D/parity_$(basename $L).log
done
for rep in 1 2 3; do for M in "300 300 300" "400 400 400"; do for L in "$@"; do
  MINIFE_LIB_PATH=$L timeout 300 python tools/ab_solve.py $M 4 >> $D/ab.jsonl 2>>$D/err.log
done; done; done
