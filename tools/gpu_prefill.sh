# prefill: parity tests on the B200
nvidia-smi -L
timeout 600 python -m pytest tests/test_prefill_gpu.py -x -q 2>&1 | tail -30 > gpurun_out/prefill_tests.log
cat gpurun_out/prefill_tests.log
