#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
MINIFE_X_LATE=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "virtual or single_gpu" > gpurun_out/gpu_tests_xl0.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_xl0.log
for n in 300 100; do
  for xl in 0 1; do
   MINIFE_X_LATE=$xl timeout 300 python tools/spmv_ab.py $n sym --parity >> gpurun_out/ab11.jsonl 2>&1
  done
done
