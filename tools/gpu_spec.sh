timeout 900 python -m pytest tests/test_stack_gpu.py tests/test_configs_gpu.py tests/test_bridge.py -x -q > gpurun_out/pytest_stack.log 2>&1; echo "rc $?" >> gpurun_out/pytest_stack.log
timeout 300 python tools/profile_stack.py --tokens 48 --allhit --timeline > gpurun_out/tl_hit.log 2>&1
timeout 300 python tools/profile_stack.py --tokens 96 --timeline > gpurun_out/tl_miss.log 2>&1
MOEB_NO_SPEC=1 timeout 300 python tools/profile_stack.py --tokens 48 --allhit --timeline > gpurun_out/tl_hit_nospec.log 2>&1
