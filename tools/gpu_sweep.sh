#!/bin/bash
mkdir -p gpurun_out/sweep
for n in 10 100 400; do
  timeout 900 python bench.py --mesh $n $n $n --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/sweep/s_${n}.log 2>&1
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/sweep/ref.log 2>&1
