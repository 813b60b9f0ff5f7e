#!/bin/bash
# quick GPU pass: build, parity + 300^3 golden tests, short bench
D=gpurun_out/${1:-quick}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -q -x -k "not 400 and not 600" > $D/gpu_tests.log 2>&1; echo "rc=$?" >> $D/gpu_tests.log
timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-format-compare > $D/bench.log 2>&1
