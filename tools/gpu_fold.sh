#!/bin/bash
D=gpurun_out/${1:-fold}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_verify.py -m gpu -q -x > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
for f in 1 0; do
  timeout 300 python tools/part_profile.py 100 100 100 4 3 --opt fold_comm=$f >> $D/parts.log 2>&1
  timeout 300 python tools/part_profile.py 400 400 400 8 3 --opt fold_comm=$f >> $D/parts.log 2>&1
  timeout 300 python tools/part_profile.py 600 300 300 2 3 --opt fold_comm=$f >> $D/parts.log 2>&1
done
timeout 300 python tools/part_profile.py 100 100 100 4 0 >> $D/parts.log 2>&1
