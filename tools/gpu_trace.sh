#!/bin/bash
# Timeline traces of solves (tools/trace_mid.py on the -DSYMM_TRACE build, which must exist:
# tools/build_flags.sh trace -DSYMM_TRACE):  tools/gpu_trace.sh OUT N1 N2 ...
D=gpurun_out/$1; shift; mkdir -p $D
export MINIFE_LIB_PATH=paper_1505_08023_b200/lib/alt_trace.so
for N in "$@"; do
  timeout 300 python tools/trace_mid.py $N >> $D/trace.jsonl 2>>$D/err.log
done
