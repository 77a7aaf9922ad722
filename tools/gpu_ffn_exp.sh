set -x
rm -f gpurun_out/ffn_exp.log
for env in "MOEB_NO_SPEC=1" "MOEB_NO_SPEC=1 MOEB_SK_UNIT=8" "MOEB_NO_SPEC=1 MOEB_SK_UNIT=16" "MOEB_NO_SPEC=1 MOEB_SK_UNIT=2" "MOEB_NO_SPEC=1 MOEB_SK_STAGES=8" "MOEB_X=0"; do
  echo "== env [$env]" >> gpurun_out/ffn_exp.log
  env $env timeout 300 python tools/profile_stack.py --tokens 24 --allhit --timeline >> gpurun_out/ffn_exp.log 2>&1
done
for b in 8 32; do
  echo "== B=$b" >> gpurun_out/ffn_exp.log
  timeout 300 python tools/profile_stack.py --tokens 12 --batch $b --allhit --timeline >> gpurun_out/ffn_exp.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
