#!/bin/bash
# A/B of the SYMM L2 policy flags (MINIFE_SYM_L2) at 400^3 and 300^3: per-launch SpMV time,
# CG iteration, and DRAM bytes of one SpMV launch (ncu, warm caches)
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for n in ${MESHES:-400 300}; do
  for f in ${FLAGS:-0 1 2 4 5 7}; do
    r=$(MINIFE_SYM_L2=$f python tools/spmv_ab.py $n sym | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['spmv_ms'],4), round(d['iter_ms'],4))")
    b=$(MINIFE_SYM_L2=$f ncu --metrics dram__bytes_read.sum --cache-control none --clock-control none -k regex:k_spmv_symm -s 20 -c 1 python tools/spmv_ab.py $n sym 2>&1 | grep dram__bytes_read | awk '{print $3 $2}')
    echo "n=$n l2=$f spmv,iter=$r dram_read=$b"
  done
done
