#!/bin/bash
# Size sweep of the default bench (one GPU): CG GFLOP/s per mesh, into gpurun_out/${1:-sweep}
D=gpurun_out/${1:-sweep}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for n in 10 20 40 60 80 100 120 150 200 250 300 400; do
  timeout 900 python bench.py --mesh $n $n $n --steps 3 --no-cpu-baseline --no-e2e --no-format-compare > $D/s_${n}.log 2>&1
done
