#!/bin/bash
# ncu captures of the update kernels and the SpMV at 300^3, and a launch list at 100^3
D=gpurun_out/${1:-prof}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 300 python tools/spmv_ab.py 300 sym > $D/ab300.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_spmv_symm" -s 120 -c 6 -o $D/upd300 python tools/spmv_ab.py 300 sym > $D/ncu_upd300.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches100.csv -s 200 -c 400 python tools/spmv_ab.py 100 sym > $D/ncu_l100.log 2>&1
timeout 300 python tools/spmv_ab.py 100 sym > $D/ab100.log 2>&1
