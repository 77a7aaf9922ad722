# prefill: per-kernel launch lists (N = 512, 4096) and full captures of the grouped GEMM
set -x
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for N in 512 4096; do
timeout 900 ncu --metrics $M --clock-control none -k regex:pf_ -c 130 --csv --log-file gpurun_out/pf_launches_$N.csv python tools/bench_prefill.py --tokens $N --capped-tokens "" --reps 1 --cpu-tokens 0 > gpurun_out/pf_ncu_$N.log 2>&1
python tools/launch_summary.py gpurun_out/pf_launches_$N.csv "prefill launch list, N=$N" "ncu ... bench_prefill.py --tokens $N" > gpurun_out/pf_launches_$N.md
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pf_gemm -s 10 -c 1 -o gpurun_out/pf_gemm_4096 python tools/bench_prefill.py --tokens 4096 --capped-tokens "" --reps 1 --cpu-tokens 0 > gpurun_out/pf_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pf_gemm -s 10 -c 1 -o gpurun_out/pf_gemm_512 python tools/bench_prefill.py --tokens 512 --capped-tokens "" --reps 1 --cpu-tokens 0 > gpurun_out/pf_full512.log 2>&1
cat gpurun_out/pf_launches_*.md
