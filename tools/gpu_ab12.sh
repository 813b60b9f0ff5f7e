#!/bin/bash
for d in 0 1 2 3; do MINIFE_SYM_DBG=$d python tools/spmv_time.py 300 sym >> gpurun_out/ab12.jsonl 2>&1; done
python tools/spmv_time.py 300 seg >> gpurun_out/ab12.jsonl 2>&1
