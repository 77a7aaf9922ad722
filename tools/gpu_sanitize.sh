# compute-sanitizer (memcheck, racecheck on the decision CTA's shared memory)
# over a small stack: the stack detects the tool and runs in serial mode
set -x
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/san_small.py > gpurun_out/sanitizer_memcheck.log 2>&1; echo "memcheck rc $?" >> gpurun_out/sanitizer_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 20 python tools/san_small.py > gpurun_out/sanitizer_racecheck.log 2>&1; echo "racecheck rc $?" >> gpurun_out/sanitizer_racecheck.log
