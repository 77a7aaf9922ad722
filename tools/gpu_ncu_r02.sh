# round-2 ncu evidence for profiles/: launch lists (miss workload — possible now
# that ncu switches the stack to its serial mode — and all-resident) and full
# captures of the hot kernels
set -x
K='regex:ffn_splitk|ffn_umma|ffn_tma|gate_decide'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" -c 208 --csv --log-file gpurun_out/launches_miss.csv python tools/profile_stack.py --tokens 6 > gpurun_out/ncu_launch_miss.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$K" -c 104 --csv --log-file gpurun_out/launches_allhit.csv python tools/profile_stack.py --tokens 4 --allhit > gpurun_out/ncu_launch_allhit.log 2>&1
MOEB_NO_SPEC=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_splitk -s 40 -c 1 -o gpurun_out/ffn_full python tools/profile_stack.py --tokens 4 --allhit > gpurun_out/ncu_ffn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gate_decide -s 40 -c 1 -o gpurun_out/gate_full python tools/profile_stack.py --tokens 4 --allhit > gpurun_out/ncu_gate.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_umma -s 20 -c 1 -o gpurun_out/umma_b8 python tools/profile_stack.py --tokens 3 --batch 8 --allhit > gpurun_out/ncu_umma.log 2>&1
ls -la gpurun_out
