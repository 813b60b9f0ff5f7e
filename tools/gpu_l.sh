#!/bin/bash
D=gpurun_out/${1:-l}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for tr in 3 0; do
python tools/part_profile.py 100 100 100 4 $tr > $D/plain_$tr.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 300 --csv --log-file $D/launches_$tr.csv python tools/part_profile.py 100 100 100 4 $tr > $D/ncu_$tr.log 2>&1
done
