# serial-mode / parity round: GPU tests, then smoke() under an ncu launch
# capture (the driver's GPUTEST shape) with a wall-clock bound
set -x
nvidia-smi -L; nproc; lscpu | grep -E "Model name|Socket|NUMA|Flags" | cut -c1-300
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
start=$(date +%s)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1
echo "smoke under ncu rc $? in $(( $(date +%s) - start )) s" >> gpurun_out/smoke_ncu.log
