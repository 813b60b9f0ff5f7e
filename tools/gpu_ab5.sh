#!/bin/bash
mkdir -p gpurun_out
for n in 300; do
  for c in 5 6; do
   MINIFE_SYM_CFG=$c timeout 300 python tools/spmv_ab.py $n sym >> gpurun_out/ab5.jsonl 2>&1
  done
done
