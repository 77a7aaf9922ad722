set -x
timeout 600 python -m pytest tests/test_moe_stack_cpp.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
C=paper_2508_18983_b200/csrc
make -C $C clean > /dev/null; make -j16 -C $C PROFILE=1 > gpurun_out/build_profile.log 2>&1
for args in "--tokens 24" "--tokens 24 --allhit" "--tokens 12 --batch 32 --allhit"; do
  echo "== $args" >> gpurun_out/phases.log
  timeout 300 python tools/profile_stack.py $args --time >> gpurun_out/phases.log 2>&1
done
make -C $C clean > /dev/null; make -j16 -C $C > gpurun_out/build.log 2>&1
