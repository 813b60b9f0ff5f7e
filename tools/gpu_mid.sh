#!/bin/bash
D=gpurun_out/${1:-mid}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for rep in 1 2; do for n in 60 100 150; do
  timeout 300 python tools/spmv_ab.py $n sym >> $D/ab.jsonl 2>>$D/err.log
  timeout 300 python tools/spmv_ab.py $n seg >> $D/ab.jsonl 2>>$D/err.log
  timeout 300 python tools/spmv_ab.py $n seg --fused >> $D/ab.jsonl 2>>$D/err.log
done; done
