#!/bin/bash
mkdir -p gpurun_out
for n in 300; do
  for d in 0 2 3 4; do
   MINIFE_GATHER=plain MINIFE_SYM_DBG=$d timeout 300 python tools/spmv_ab.py $n sym >> gpurun_out/ab2.jsonl 2>&1
  done
  MINIFE_GATHER=plain MINIFE_SYM_DBG=3 MINIFE_SYM_CFG=2 timeout 300 python tools/spmv_ab.py $n sym >> gpurun_out/ab2.jsonl 2>&1
done
