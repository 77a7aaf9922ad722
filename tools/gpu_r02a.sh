set -x
timeout 600 python -m pytest tests/test_moe_stack_cpp.py tests/test_stack_gpu.py -k "cpp or serial" -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
start=$(date +%s)
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1
echo "smoke under ncu rc $? in $(( $(date +%s) - start )) s" >> gpurun_out/smoke_ncu.log
bash tools/gpu_phases.sh
