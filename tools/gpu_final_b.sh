# round-end evidence, part B: every named config at 1 GPU and prefill TTFT
set -x
timeout 2400 python tools/bench_configs.py --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1; echo "configs rc $?" >> gpurun_out/configs.log
timeout 900 python tools/bench_prefill.py --out gpurun_out/prefill.json > gpurun_out/prefill.log 2>&1; echo "prefill rc $?" >> gpurun_out/prefill.log
