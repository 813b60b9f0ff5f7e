#!/bin/bash
# Parity of the L2-reuse options, then an interleaved A/B at mid-size (tools/ab_solve.py)
D=gpurun_out/$1; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "other_options or band_order" > $D/tests.log 2>&1; echo rc=$? >> $D/tests.log
for rep in 1 2; do for N in 100 150; do
  for O in "snake=0" "snake=1" "snake=1 --opt val_evict_first=0" "l2_pin_mb=40" "l2_pin_mb=70" "l2_pin_mb=100" "l2_pin_mb=70 --opt val_evict_first=0"; do
    timeout 300 python tools/ab_solve.py $N $N $N 2 --opt $O >> $D/ab.jsonl 2>>$D/err.log
  done
done; done
