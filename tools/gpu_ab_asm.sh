#!/bin/bash
D=gpurun_out/$1; N=$2; shift 2; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for rep in 1 2 3; do for L in "$@"; do MINIFE_LIB_PATH=$L timeout 120 python tools/ab_asm.py $N >> $D/ab.jsonl 2>>$D/err.log; done; done
