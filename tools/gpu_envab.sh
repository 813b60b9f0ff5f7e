#!/bin/bash
# A/B of one MINIFE_* environment toggle: ENVVAR=NAME VALUES="a b c" MESHES="300 100"
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for n in ${MESHES:-300 100}; do
  for v in ${VALUES}; do
    env $ENVVAR=$v python tools/spmv_ab.py $n sym | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('n=$n $ENVVAR=$v spmv', round(d['spmv_ms'],4), 'upd', round(d['upd_ms'],4), 'iter', round(d['iter_ms'],4))"
  done
done
