#!/bin/bash
D=gpurun_out/${1:-repro}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "band or option" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
for cfg in "400 1 1 -1" "400 0 0 -1" "300 1 1 -1"; do
  echo "== $cfg" >> $D/out.log
  timeout 300 python tools/repro400.py $cfg >> $D/out.log 2>&1; echo "rc=$?" >> $D/out.log
done
timeout 900 python bench.py --mesh 400 400 400 --steps 3 --no-cpu-baseline --no-e2e > $D/sweep_400.log 2>&1; echo "rc=$?" >> $D/sweep_400.log
