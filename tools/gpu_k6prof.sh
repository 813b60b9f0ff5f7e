#!/bin/bash
# ncu source-level capture of K6 and the SpMV at one mesh: tools/gpu_k6prof.sh OUT N
D=gpurun_out/$1; N=${2:-100}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 300 python tools/spmv_ab.py $N sym > $D/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_update_xr|k_spmv_symm|k_update_p" -s 400 -c 3 -o $D/mid$N python tools/spmv_ab.py $N sym > $D/ncu.log 2>&1
echo rc=$? >> $D/ncu.log
