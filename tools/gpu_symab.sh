#!/bin/bash
# A/B of SYM SpMV kernel configurations (MINIFE_SYM_CFG): per-launch SpMV time at 300^3 and
# 100^3 with a partition-independence check per run; optional full GPU suite per config
mkdir -p gpurun_out/ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab/build.log 2>&1 || exit 1
OUT=gpurun_out/ab/${TAG:-ab}.jsonl
for c in ${CFGS:-1}; do
  for n in ${MESHES:-300 100}; do
    MINIFE_SYM_CFG=$c timeout 300 python tools/spmv_ab.py $n sym --parity >> $OUT 2>>gpurun_out/ab/err.log
  done
done
for c in ${TESTCFGS:-}; do
  MINIFE_SYM_CFG=$c timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab/tests_cfg$c.log 2>&1
  echo "cfg $c: $(tail -1 gpurun_out/ab/tests_cfg$c.log)"
done
python - "$OUT" <<'PY'
import sys, json
for l in open(sys.argv[1]):
    d = json.loads(l)
    print(d['n'], d['env'].get('MINIFE_SYM_CFG', '-'), round(d['spmv_ms'], 4), round(d['upd_ms'], 4),
          round(d['iter_ms'], 4), d.get('parity_vs_virtual2'))
PY
tail -3 gpurun_out/ab/err.log
