#!/bin/bash
D=gpurun_out/${1:-band}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_golden.py -m gpu -q -x -k "400cubed_single or 300cubed_bench" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
for rep in 1 2; do for b in 0 65536 98304 131072; do
  timeout 300 python tools/ab_solve.py 400 400 400 4 --opt band_rows=$b >> $D/ab.jsonl 2>>$D/err.log
done; done
for b in 0 98304; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_spmv_symm -s 100 -c 2 --csv python tools/spmv_ab.py 400 sym --opt band_rows=$b > $D/ncu_$b.csv 2>>$D/err.log
done
