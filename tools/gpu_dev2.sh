#!/bin/bash
D=gpurun_out/${1:-dev}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for rep in 1 2; do for o in "x_defer=0" "x_defer=-1"; do
  timeout 300 python tools/part_profile.py 600 300 300 2 3 --opt $o >> $D/parts.log 2>&1
  timeout 300 python tools/part_profile.py 600 300 300 2 0 --opt $o >> $D/parts.log 2>&1
  timeout 300 python tools/part_profile.py 400 400 400 8 3 --opt $o >> $D/parts.log 2>&1
  timeout 300 python tools/part_profile.py 400 400 400 8 0 --opt $o >> $D/parts.log 2>&1
done; done
