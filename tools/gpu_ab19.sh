#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for n in 300 100 40; do
  for pdl in 0 1; do
   MINIFE_PDL=$pdl timeout 200 python tools/spmv_ab.py $n sym --parity >> gpurun_out/ab19.jsonl 2>&1 || echo "n $n pdl $pdl failed" >> gpurun_out/ab19.jsonl
  done
done
