timeout 900 python -m pytest tests -m gpu -q -x -k "not slow" > gpurun_out/gpu_tests12.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests12.log
for m in "10 10 10" "100 100 100"; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-format-compare --mesh $m > "gpurun_out/sweep12_${m// /x}.log" 2>&1; done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-format-compare > gpurun_out/bench12.log 2>&1
