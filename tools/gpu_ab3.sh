#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for n in 10 100 300; do
  timeout 300 python tools/spmv_ab.py $n sym >> gpurun_out/ab3.jsonl 2>&1
  timeout 300 python tools/spmv_ab.py $n seg >> gpurun_out/ab3.jsonl 2>&1
done
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
