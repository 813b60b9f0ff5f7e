timeout 1500 python -m pytest tests -m gpu -q -x -k "not slow" > gpurun_out/gpu_tests23.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests23.log
for m in "10 10 10" "100 100 100" "300 300 300" "400 400 400"; do timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --mesh $m > "gpurun_out/s23_${m// /x}.log" 2>&1; done
