#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for n in 300 100 40; do
   timeout 200 python tools/spmv_ab.py $n sym >> gpurun_out/ab22.jsonl 2>&1 || echo "n $n failed" >> gpurun_out/ab22.jsonl
done
timeout 200 python tools/spmv_ab.py 100 seg >> gpurun_out/ab22.jsonl 2>&1
