# round-end evidence, part A: GPU tests, smoke, the bench line, the reference
# arm, per-upload PCIe rates, ncu launch lists and full captures of the hot
# kernels (each ncu command only after the same command ran clean without it)
set -x
nvidia-smi -L; nproc
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo "ref rc $?" >> gpurun_out/bench_ref.log
timeout 300 python tools/profile_stack.py --tokens 64 --uploads > gpurun_out/uploads.log 2>&1
timeout 300 python tools/ffn_phases.py --allhit --tokens 24 > gpurun_out/ffn_phases_allhit.log 2>&1
timeout 300 python tools/ffn_phases.py --tokens 24 > gpurun_out/ffn_phases_miss.log 2>&1
K='regex:ffn_splitk|ffn_umma|ffn_tma|gate_decide'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" -c 208 --csv --log-file gpurun_out/launches_miss.csv python tools/profile_stack.py --tokens 6 > gpurun_out/ncu_launch_miss.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" -c 104 --csv --log-file gpurun_out/launches_allhit.csv python tools/profile_stack.py --tokens 4 --allhit > gpurun_out/ncu_launch_allhit.log 2>&1
MOEB_NO_SPEC=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_splitk -s 40 -c 1 -o gpurun_out/ffn_full python tools/profile_stack.py --tokens 4 --allhit > gpurun_out/ncu_ffn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gate_decide -s 40 -c 1 -o gpurun_out/gate_full python tools/profile_stack.py --tokens 4 --allhit > gpurun_out/ncu_gate.log 2>&1
ls -la gpurun_out
