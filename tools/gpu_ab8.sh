#!/bin/bash
mkdir -p gpurun_out
MINIFE_SYM_CFG=6 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_cfg6.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests_cfg6.log
for n in 300 100 10; do
  for c in 0 6 7; do
   MINIFE_SYM_CFG=$c timeout 300 python tools/spmv_ab.py $n sym >> gpurun_out/ab8.jsonl 2>&1
  done
done
