#!/bin/bash
# Parity of the working tree (exact-dot and parity suites), trace, interleaved A/B vs HEAD
D=gpurun_out/$1; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dot.py tests/test_gpu_parity.py -m gpu -x -q > $D/tests.log 2>&1; echo rc=$? >> $D/tests.log
MINIFE_LIB_PATH=paper_1505_08023_b200/lib/alt_trace.so timeout 300 python tools/trace_mid.py 100 >> $D/trace.jsonl 2>>$D/err.log
for rep in 1 2; do for N in 60 100 300; do for L in base flushnew; do
  MINIFE_LIB_PATH=paper_1505_08023_b200/lib/alt_$L.so timeout 300 python tools/ab_solve.py $N $N $N 3 >> $D/ab.jsonl 2>>$D/err.log
done; done; done
