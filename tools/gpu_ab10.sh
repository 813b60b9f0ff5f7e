#!/bin/bash
mkdir -p gpurun_out
for n in 300 100; do
  for c in 0 1 2 3; do
   MINIFE_SYM_CFG=$c timeout 300 python tools/spmv_ab.py $n sym --parity >> gpurun_out/ab10.jsonl 2>&1
  done
done
