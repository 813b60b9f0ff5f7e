#!/bin/bash
D=gpurun_out/${1:-band}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for rep in 1 2; do for M in "300 300 300" "400 400 400"; do for b in 0 24576 49152 65536; do
  timeout 300 python tools/ab_solve.py $M 4 --opt band_rows=$b >> $D/ab.jsonl 2>>$D/err.log
done; done; done
for b in 49152 65536; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_spmv_symm -s 100 -c 2 --csv python tools/spmv_ab.py 400 sym --opt band_rows=$b > $D/ncu400_$b.csv 2>>$D/err.log
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_spmv_symm -s 100 -c 2 --csv python tools/spmv_ab.py 300 sym --opt band_rows=$b > $D/ncu300_$b.csv 2>>$D/err.log
done
