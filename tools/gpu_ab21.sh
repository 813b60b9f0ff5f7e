#!/bin/bash
mkdir -p gpurun_out
for c in 1 2 3 4; do
  MINIFE_SYM_CFG=$c timeout 200 python tools/spmv_ab.py 300 sym >> gpurun_out/ab21.jsonl 2>&1 || echo "cfg $c failed" >> gpurun_out/ab21.jsonl
  MINIFE_SYM_CFG=$c timeout 200 python tools/spmv_ab.py 100 sym --parity >> gpurun_out/ab21.jsonl 2>&1 || echo "cfg $c failed" >> gpurun_out/ab21.jsonl
done
