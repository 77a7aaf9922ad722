set -x
C=paper_2508_18983_b200/csrc
rm -f gpurun_out/phases.log
make -C $C clean > /dev/null; make -j16 -C $C PROFILE=1 > gpurun_out/build_profile.log 2>&1
for args in "--tokens 48" "--tokens 24 --allhit"; do
  echo "== PROFILE $args --timeline" >> gpurun_out/phases.log
  timeout 300 python tools/profile_stack.py $args --timeline >> gpurun_out/phases.log 2>&1
done
make -C $C clean > /dev/null; make -j16 -C $C > gpurun_out/build.log 2>&1
echo "== uploads" >> gpurun_out/phases.log
timeout 300 python tools/profile_stack.py --tokens 64 --uploads >> gpurun_out/phases.log 2>&1
./tools/probe/pcie_probe > gpurun_out/pcie_probe.txt 2>&1
