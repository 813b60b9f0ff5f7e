#!/bin/bash
mkdir -p gpurun_out
for c in 2 4; do
  MINIFE_SYM_CFG=$c timeout 200 python tools/spmv_ab.py 300 sym >> gpurun_out/ab14.jsonl 2>&1 || echo "cfg $c failed" >> gpurun_out/ab14.jsonl
  MINIFE_SYM_CFG=$c timeout 120 python tools/spmv_time.py 300 sym >> gpurun_out/ab14.jsonl 2>&1 || echo "cfg $c t300 failed" >> gpurun_out/ab14.jsonl
done
