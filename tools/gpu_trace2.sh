#!/bin/bash
D=gpurun_out/$1; shift; mkdir -p $D
export MINIFE_LIB_PATH=paper_1505_08023_b200/lib/alt_trace.so
for N in "$@"; do
  timeout 300 python tools/trace_mid.py $N >> $D/trace.jsonl 2>>$D/err.log
done
