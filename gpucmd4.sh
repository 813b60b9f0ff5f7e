timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests4.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests4.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.log 2>&1; echo "bench exit $?" >> gpurun_out/bench4.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --format crs --no-e2e > gpurun_out/bench4crs.log 2>&1; echo "bench exit $?" >> gpurun_out/bench4crs.log
