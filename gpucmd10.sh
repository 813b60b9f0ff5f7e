timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests10.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests10.log
for m in "10 10 10" "100 100 100" "400 400 400"; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --mesh $m > "gpurun_out/sweep_${m// /x}.log" 2>&1; done
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench10.log 2>&1; echo "bench exit $?" >> gpurun_out/bench10.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-format-compare > gpurun_out/bench10_torchrun.log 2>&1; echo "torchrun exit $?" >> gpurun_out/bench10_torchrun.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench10_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/bench10_ref.log
