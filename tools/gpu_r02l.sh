set -x
rm -f gpurun_out/phases.log
for args in "--tokens 48" "--tokens 48 --shape qwen --layers 24" "--tokens 24 --shape qwen --layers 24 --allhit"; do
  echo "== $args --timeline" >> gpurun_out/phases.log
  timeout 300 python tools/profile_stack.py $args --timeline >> gpurun_out/phases.log 2>&1
done
timeout 600 python tools/bench_configs.py --only C2P --no-cpu --out gpurun_out/c2p.json > gpurun_out/c2p.log 2>&1
