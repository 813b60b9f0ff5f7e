#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for n in 10 15 19; do
  for sm in 0 1 2; do
   MINIFE_SMALL=$sm timeout 120 python tools/spmv_ab.py $n sym --parity >> gpurun_out/ab17.jsonl 2>&1 || echo "n $n sm $sm failed" >> gpurun_out/ab17.jsonl
  done
done
