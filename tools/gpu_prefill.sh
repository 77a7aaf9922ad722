# prefill: parity tests, TTFT, launch list and a full capture of the grouped GEMM
nvidia-smi -L
timeout 600 python -m pytest tests/test_prefill_gpu.py -x -q 2>&1 | tail -30 > gpurun_out/prefill_tests.log
cat gpurun_out/prefill_tests.log
timeout 900 python tools/bench_prefill.py --cpu-tokens 0 --out gpurun_out/prefill.json 2>&1 | tail -20
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for N in 512 4096; do
timeout 900 ncu --metrics $M --clock-control none -k regex:pf_ -c 130 --csv --log-file gpurun_out/pf_launches_$N.csv python tools/bench_prefill.py --tokens $N --capped-tokens "" --reps 1 --cpu-tokens 0 > gpurun_out/pf_ncu_$N.log 2>&1
python tools/launch_summary.py gpurun_out/pf_launches_$N.csv "prefill launch list, N=$N" "ncu ... bench_prefill.py --tokens $N" > gpurun_out/pf_launches_$N.md
done
cat gpurun_out/pf_launches_*.md
