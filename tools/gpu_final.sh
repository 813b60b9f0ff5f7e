#!/bin/bash
# Full evidence pass: tests, smoke, bench (+reference arm), sweep, ncu launch list + capture.
D=gpurun_out/${1:-final}; mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $D/smi.txt
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $D/gpu_tests.log 2>&1; echo "tests rc=$?" >> $D/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 900 python bench.py > $D/bench.log 2>&1; echo "bench rc=$?" >> $D/bench.log
timeout 900 python bench.py > $D/bench_repeat.log 2>&1
timeout 600 python bench.py --impl reference > $D/bench_ref.log 2>&1
for n in 10 100 400; do
  timeout 900 python bench.py --mesh $n $n $n --steps 3 --no-cpu-baseline --no-e2e > $D/sweep_${n}.log 2>&1
done
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-format-compare"
$B > $D/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1300 --csv --log-file $D/launches.csv $B > $D/ncu_launch.log 2>&1
timeout 300 python tools/spmv_ab.py 300 sym > $D/plain_ab.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_spmv_symm|k_update|k_assemble" -s 60 -c 4 -o $D/hot300 python tools/spmv_ab.py 300 sym > $D/ncu_full.log 2>&1
