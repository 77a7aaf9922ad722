set -x
nvidia-smi -L; lscpu | head -20
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python tools/profile_stack.py --tokens 8 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn -s 20 -c 1 -o gpurun_out/ffn python tools/profile_stack.py --tokens 4 --allhit > gpurun_out/ncu_ffn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gate_decide -s 20 -c 1 -o gpurun_out/gate python tools/profile_stack.py --tokens 4 --allhit > gpurun_out/ncu_gate.log 2>&1
ls -la gpurun_out
