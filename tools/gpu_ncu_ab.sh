#!/bin/bash
# Same-box ncu A/B of SpMV launch time for library variants: tools/gpu_ncu_ab.sh OUT N libA libB ...
D=gpurun_out/$1; N=$2; shift 2; mkdir -p $D
for rep in 1 2; do for L in "$@"; do
  MINIFE_LIB_PATH=paper_1505_08023_b200/lib/alt_$L.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__registers_per_thread --clock-control none -k regex:"k_spmv_symm" -s 60 -c 8 --csv python tools/spmv_ab.py $N sym > $D/ncu_${L}_$rep.csv 2>&1
done; done
