# headline bench + every named config at 1 GPU + the reference arm
set -x
nvidia-smi -L; nproc
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo "ref rc $?" >> gpurun_out/bench_ref.log
timeout 2400 python tools/bench_configs.py --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1; echo "configs rc $?" >> gpurun_out/configs.log
