#!/bin/bash
# One GPU call: build, parity tests, smoke, default bench (into gpurun_out/$1, default "check").
D=gpurun_out/${1:-check}
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $D/smi.txt
free -g >> $D/smi.txt
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > $D/gpu_tests.log 2>&1; echo "tests rc=$?" >> $D/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 900 python bench.py > $D/bench.log 2>&1; echo "bench rc=$?" >> $D/bench.log
