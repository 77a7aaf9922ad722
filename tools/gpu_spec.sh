set -x
timeout 900 python -m pytest tests/test_stack_gpu.py tests/test_configs_gpu.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/phases.log
for env in "MOEB_X=0" "MOEB_SPEC_UPLOAD=0"; do
  echo "== $env --tokens 64 --timeline" >> gpurun_out/phases.log
  env $env timeout 300 python tools/profile_stack.py --tokens 64 --timeline >> gpurun_out/phases.log 2>&1
done
timeout 900 python bench.py --no-cpu-baseline --no-batched --no-c5 > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
