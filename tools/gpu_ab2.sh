#!/bin/bash
# Interleaved A/B of library builds at 300^3 and 400^3 + ncu DRAM bytes of one SpMV launch
# at 400^3 per build:  tools/gpu_ab2.sh OUT libA.so libB.so ...
D=gpurun_out/$1; shift; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for rep in 1 2; do for M in "300 300 300" "400 400 400"; do for L in "$@"; do
  MINIFE_LIB_PATH=$L timeout 300 python tools/ab_solve.py $M 4 >> $D/ab.jsonl 2>>$D/err.log
done; done; done
for L in "$@"; do
  MINIFE_LIB_PATH=$L timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_spmv_symm -s 100 -c 2 --csv python tools/spmv_ab.py 400 sym > $D/ncu_$(basename $L).csv 2>>$D/err.log
done
