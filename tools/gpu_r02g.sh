set -x
bash tools/gpu_phases.sh
timeout 600 python -m pytest tests/test_stack_gpu.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
