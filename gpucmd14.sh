timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests14.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests14.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-format-compare > gpurun_out/bench14.log 2>&1
