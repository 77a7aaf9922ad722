set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-batched --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
