#!/bin/bash
D=gpurun_out/$1; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dot.py tests/test_gpu_parity.py -m gpu -x -q > $D/tests.log 2>&1; echo rc=$? >> $D/tests.log
for rep in 1 2; do for N in 80 100 120; do for O in snake=0 snake=1; do
  timeout 300 python tools/ab_solve.py $N $N $N 3 --opt $O >> $D/ab.jsonl 2>>$D/err.log
done; done; done
