set -x
rm -f gpurun_out/phases.log
for args in "--tokens 48" "--tokens 24 --allhit"; do
  echo "== $args --timeline" >> gpurun_out/phases.log
  timeout 300 python tools/profile_stack.py $args --timeline >> gpurun_out/phases.log 2>&1
done
timeout 900 python bench.py --no-cpu-baseline --no-batched --no-c5 > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
timeout 600 python -m pytest tests/test_stack_gpu.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
