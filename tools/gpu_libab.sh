#!/bin/bash
# tw_drift for the default library and alternative builds in lib/alt_*.so
mkdir -p gpurun_out/libab
python tools/tw_drift.py ${N:-300} > gpurun_out/libab/default.json 2>&1
for f in paper_1505_08023_b200/lib/alt_*.so; do
  b=$(basename $f .so)
  MINIFE_LIB_PATH=$PWD/$f python tools/tw_drift.py ${N:-300} > gpurun_out/libab/$b.json 2>&1
done
for f in gpurun_out/libab/*.json; do
  python -c "
import json,sys; d=json.loads(open('$f').read()); w=d['window_spmv_iter_avg_ms']
print('$f'.split('/')[-1], 'solve avg', round(sum(v[2] for r in w.values() for v in r)/sum(len(r) for r in w.values()),4), {k: (r[1][0], r[1][1]) for k,r in w.items()})"
done
