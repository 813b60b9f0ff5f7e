#!/bin/bash
mkdir -p gpurun_out
for c in 0 4; do
  for lib in default _libs/nexp2.so _libs/nexp3.so; do
    if [ "$lib" = default ]; then L=""; else L="$PWD/$lib"; fi
    MINIFE_LIB_PATH=$L MINIFE_SYM_CFG=$c timeout 200 python tools/spmv_ab.py 300 sym >> gpurun_out/ab15.jsonl 2>&1 || echo "cfg $c $lib failed" >> gpurun_out/ab15.jsonl
    echo "lib=$lib" >> gpurun_out/ab15.jsonl
  done
done
