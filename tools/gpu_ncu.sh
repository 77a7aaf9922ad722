# ncu evidence for profiles/: launch list of the timed workload shape + full captures of the hot kernels
set -x
# launch list: skip the weight-synthesis launches (26*64*3 + ...), capture 2 tokens of the miss workload
# (miss mode cannot run under ncu: kernel serialisation stalls the copy stream the FFN waits on)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"ffn_splitk|ffn_tma|gate_decide" -c 104 --csv --log-file gpurun_out/launches_allhit.csv python tools/profile_stack.py --tokens 4 --allhit > gpurun_out/ncu_launch2.log 2>&1
MOEB_NO_SPEC=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_splitk|ffn_tma" -s 40 -c 1 -o gpurun_out/ffn_full python tools/profile_stack.py --tokens 4 --allhit > gpurun_out/ncu_ffn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gate_decide -s 40 -c 1 -o gpurun_out/gate_full python tools/profile_stack.py --tokens 4 --allhit > gpurun_out/ncu_gate.log 2>&1
ls -la gpurun_out
