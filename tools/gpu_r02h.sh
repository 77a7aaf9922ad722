set -x
rm -f gpurun_out/phases.log
for env in "MOEB_X=0" "MOEB_NO_SHARED_FIRST=1"; do
for args in "--tokens 48" "--tokens 24 --allhit"; do
  echo "== $env $args --timeline" >> gpurun_out/phases.log
  env $env timeout 300 python tools/profile_stack.py $args --timeline >> gpurun_out/phases.log 2>&1
done
done
timeout 600 python -m pytest tests/test_stack_gpu.py tests/test_predictor_gpu.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
