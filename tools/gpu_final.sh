#!/bin/bash
# Full evidence pass: tests, smoke, bench (+reference arm), sweep, ncu launch list + captures.
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/final/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.log
timeout 900 python bench.py > gpurun_out/final/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/final/bench.log
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_ref.log 2>&1
for n in 10 100 400; do
  timeout 900 python bench.py --mesh $n $n $n --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/final/sweep_${n}.log 2>&1
done
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-format-compare"
$B > gpurun_out/final/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/final/launches.csv $B > gpurun_out/final/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_spmv_symm|k_update" -s 60 -c 3 -o gpurun_out/final/hot300 python tools/spmv_ab.py 300 sym > gpurun_out/final/ncu_full.log 2>&1
