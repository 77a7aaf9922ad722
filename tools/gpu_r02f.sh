set -x
rm -f gpurun_out/phases.log
for args in "--tokens 48" "--tokens 24 --allhit" "--tokens 12 --batch 8 --allhit" "--tokens 12 --batch 32 --allhit"; do
  echo "== $args --timeline" >> gpurun_out/phases.log
  timeout 300 python tools/profile_stack.py $args --timeline >> gpurun_out/phases.log 2>&1
done
timeout 900 python -m pytest tests/test_stack_gpu.py tests/test_configs_gpu.py tests/test_predictor_gpu.py -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
MOEB_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 5 --no-ablation > gpurun_out/bench_2rank.log 2>&1; echo "2rank rc $?" >> gpurun_out/bench_2rank.log
