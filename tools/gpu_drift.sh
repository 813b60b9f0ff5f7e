#!/bin/bash
# SpMV / iteration time at several positions inside the 300^3 and 400^3 solves (+ optional tests)
D=gpurun_out/${1:-drift}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 300 python tools/tw_drift.py 300 > $D/drift300.log 2>&1
timeout 300 python tools/tw_drift.py 400 > $D/drift400.log 2>&1
if [ -n "$2" ]; then timeout 1500 python -m pytest tests -m gpu -q -x > $D/gpu_tests.log 2>&1; echo "rc=$?" >> $D/gpu_tests.log; fi
