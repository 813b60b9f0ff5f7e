#!/bin/bash
# Parity of the working tree (exact-dot + parity suites), then an interleaved A/B of library
# builds: tools/gpu_ab_libs.sh OUT "N1 N2 .." libA libB ...  (names of lib/alt_NAME.so)
D=gpurun_out/$1; SIZES=$2; shift 2; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dot.py tests/test_gpu_parity.py -m gpu -x -q > $D/tests.log 2>&1; echo rc=$? >> $D/tests.log
for rep in 1 2; do for N in $SIZES; do for L in "$@"; do
  MINIFE_LIB_PATH=paper_1505_08023_b200/lib/alt_$L.so timeout 300 python tools/ab_solve.py $N $N $N 3 >> $D/ab.jsonl 2>>$D/err.log
done; done; done
