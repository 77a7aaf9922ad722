set -x
./tools/ffn_microbench 0 0 > gpurun_out/mb.log 2>&1
./tools/ffn_microbench 0 1 >> gpurun_out/mb.log 2>&1
./tools/ffn_microbench 0 2 >> gpurun_out/mb.log 2>&1
timeout 600 python -m pytest tests/test_stack_gpu.py -x -q > gpurun_out/pytest_stack.log 2>&1
timeout 300 python tools/profile_stack.py --tokens 64 --allhit --time > gpurun_out/allhit.log 2>&1
timeout 300 python tools/profile_stack.py --tokens 64 --time > gpurun_out/miss.log 2>&1
