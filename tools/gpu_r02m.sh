set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
rm -f gpurun_out/phases.log
for args in "--tokens 48" "--tokens 24 --allhit" "--tokens 12 --batch 8 --allhit" "--tokens 12 --batch 32 --allhit"; do
  echo "== $args --timeline" >> gpurun_out/phases.log
  timeout 300 python tools/profile_stack.py $args --timeline >> gpurun_out/phases.log 2>&1
done
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 20 python tools/san_small.py > gpurun_out/sanitizer_racecheck.log 2>&1 || true
