#!/bin/bash
# Why is the band tile order slower at equal DRAM bytes?  ncu --set full of one in-solve SYM
# SpMV at 300^3 natural / banded and 400^3 banded / natural: tools/gpu_band_prof.sh OUT
D=gpurun_out/${1:-bandprof}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for cfg in "300 0" "300 65536" "400 65536" "400 0"; do
  set -- $cfg
  timeout 300 python tools/spmv_ab.py $1 sym --opt band_rows=$2 >> $D/times.jsonl 2>>$D/err.log
done
for cfg in "300 0" "300 65536" "400 65536" "400 0"; do
  set -- $cfg
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_spmv_symm" -s 60 -c 1 \
    -o $D/symm_${1}_band$2 python tools/spmv_ab.py $1 sym --opt band_rows=$2 > $D/ncu_${1}_$2.log 2>&1
  echo "$cfg rc=$?" >> $D/ncu_rc.log
done
