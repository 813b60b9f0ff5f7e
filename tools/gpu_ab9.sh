#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for n in 10 12; do
  for sm in 0 1; do
   for f in sym seg; do
   MINIFE_SMALL=$sm timeout 300 python tools/spmv_ab.py $n $f --parity >> gpurun_out/ab9.jsonl 2>&1
   done
  done
done
