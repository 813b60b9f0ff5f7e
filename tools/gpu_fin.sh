#!/bin/bash
D=gpurun_out/$1; mkdir -p $D
MINIFE_LIB_PATH=paper_1505_08023_b200/lib/alt_trace.so timeout 300 python tools/trace_mid.py 100 >> $D/trace.jsonl 2>>$D/err.log
bash tools/gpu_ab_libs.sh $1 "${2:-60 100}" head ${3:-fin}
