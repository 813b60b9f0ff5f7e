#!/bin/bash
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-format-compare"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_sym300.csv $B > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_update" -s 40 -c 2 -o gpurun_out/upd300 python tools/spmv_ab.py 300 sym > gpurun_out/ncu_upd.log 2>&1
