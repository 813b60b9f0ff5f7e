#!/bin/bash
mkdir -p gpurun_out
for c in 1 2 3; do
  MINIFE_SYM_CFG=$c timeout 120 python tools/spmv_ab.py 10 sym --parity >> gpurun_out/ab13.jsonl 2>&1 || echo "cfg $c n10 failed rc=$?" >> gpurun_out/ab13.jsonl
done
for c in 0 1 2 3; do
  MINIFE_SYM_CFG=$c timeout 120 python tools/spmv_ab.py 100 sym --parity >> gpurun_out/ab13.jsonl 2>&1 || echo "cfg $c n100 failed" >> gpurun_out/ab13.jsonl
  MINIFE_SYM_CFG=$c timeout 120 python tools/spmv_time.py 300 sym >> gpurun_out/ab13.jsonl 2>&1 || echo "cfg $c t300 failed" >> gpurun_out/ab13.jsonl
done
