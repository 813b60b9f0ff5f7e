#!/bin/bash
D=gpurun_out/${1:-p100}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_spmv_symm" -s 300 -c 3 -o $D/hot100 python tools/spmv_ab.py 100 sym > $D/ncu.log 2>&1
