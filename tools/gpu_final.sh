# round-end evidence: GPU tests, smoke, the bench line, the reference arm, every named config, prefill TTFT
set -x
nvidia-smi -L; nproc
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo "ref rc $?" >> gpurun_out/bench_ref.log
timeout 2400 python tools/bench_configs.py --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1; echo "configs rc $?" >> gpurun_out/configs.log
timeout 900 python tools/bench_prefill.py --out gpurun_out/prefill.json > gpurun_out/prefill.log 2>&1; echo "prefill rc $?" >> gpurun_out/prefill.log
timeout 300 python tools/profile_stack.py --tokens 64 --uploads > gpurun_out/uploads.log 2>&1
