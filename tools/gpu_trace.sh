#!/bin/bash
# Timeline traces of mid-size solves (tools/trace_mid.py on the -DSYMM_TRACE build)
D=gpurun_out/$1; shift; mkdir -p $D
export MINIFE_LIB_PATH=paper_1505_08023_b200/lib/alt_trace.so
for N in "$@"; do
  timeout 300 python tools/trace_mid.py $N >> $D/trace.jsonl 2>>$D/err.log
  timeout 300 python tools/trace_mid.py $N --opt snake=1 >> $D/trace.jsonl 2>>$D/err.log
done
unset MINIFE_LIB_PATH
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for O in "snake=0" "snake=1" "l2_pin_mb=70" "l2_pin_mb=70 --opt val_evict_first=0"; do
  T=$(echo $O | tr -c 'a-z0-9_\n' '_')
  timeout 600 ncu --cache-control none --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    -k regex:k_spmv_symm -s 500 -c 6 --csv python tools/spmv_ab.py 100 sym --opt $O > $D/ncu_$T.csv 2>$D/ncu_$T.err
done
