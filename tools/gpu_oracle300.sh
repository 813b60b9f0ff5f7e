#!/bin/bash
# The oracle at the headline config on the GPU box's host (1 core): full 200-iteration 300^3
# solve, timed, and its output compared with the committed golden reference
D=gpurun_out/${1:-oracle300}; mkdir -p $D
lscpu > $D/lscpu.txt 2>&1; free -g >> $D/lscpu.txt
python -c "import oracle; oracle.build()" > $D/build.log 2>&1
taskset -c 0 timeout 1500 python tools/make_golden.py 300 300 300 --out $D/minife_300x300x300.json > $D/make_golden.log 2>&1; echo "rc=$?" >> $D/make_golden.log
python - > $D/compare.txt 2>&1 <<'PY'
import json
a = json.load(open('tests/golden/minife_300x300x300.json'))
b = json.load(open('gpurun_out/oracle300/minife_300x300x300.json'))
print("sha256 identical:", a["sha256"] == b["sha256"])
print("history identical:", a["cg"]["hist_hex"] == b["cg"]["hist_hex"])
print("oracle wall s (GPU host):", b["oracle_wall_s"])
print("oracle wall s (dev host):", a["oracle_wall_s"])
PY
