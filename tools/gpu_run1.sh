#!/bin/bash
mkdir -p gpurun_out/s3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s3/build.log 2>&1 || exit 1
for n in 300 100; do timeout 300 python tools/spmv_ab.py $n sym --parity >> gpurun_out/s3/ab.jsonl 2>>gpurun_out/s3/ab.err; done
cat gpurun_out/s3/ab.jsonl; cat gpurun_out/s3/ab.err | tail -3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s3/tests.log 2>&1; tail -2 gpurun_out/s3/tests.log
timeout 600 python bench.py > gpurun_out/s3/bench.log 2>&1; tail -1 gpurun_out/s3/bench.log | cut -c1-600
