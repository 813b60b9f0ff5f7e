#!/bin/bash
# ncu source-level captures of the SYM SpMV at iteration 51 and 181 of a 300^3 solve
D=gpurun_out/${1:-late}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 300 python tools/one_solve.py 300 > $D/plain.log 2>&1 || exit 1
for K in 51 181; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmv_symm \
    -s $((K - 1)) -c 1 -o $D/spmv300_k$K python tools/one_solve.py 300 > $D/ncu_k$K.log 2>&1
done
