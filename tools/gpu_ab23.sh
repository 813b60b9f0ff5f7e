#!/bin/bash
for n in 300 100; do timeout 200 python tools/spmv_ab.py $n sym --parity >> gpurun_out/ab23.jsonl 2>&1; done
