set -x
timeout 900 python -m pytest tests/test_stack_gpu.py tests/test_predictor_gpu.py tests/test_moe_stack_cpp.py -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
