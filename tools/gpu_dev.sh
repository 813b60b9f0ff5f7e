#!/bin/bash
D=gpurun_out/${1:-dev}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -q -x -k "device or virtual or rank or weak_scaling_600x300x300 or deferred" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
for tr in 0 3; do
  timeout 300 python tools/part_profile.py 600 300 300 2 $tr >> $D/parts.log 2>&1
  timeout 300 python tools/part_profile.py 400 400 400 8 $tr >> $D/parts.log 2>&1
done
