set -u
mkdir -p gpurun_out/ab10
IFA_B200_LIB=build/corr16/libifa_b200.so timeout 300 python -m pytest "tests/test_gpu_parity.py::test_fast_mode_within_tolerance" tests/test_gpu_dump.py -q -x --timeout 60 > gpurun_out/ab10/pytest_quick.log 2>&1
echo "rc $?" >> gpurun_out/ab10/pytest_quick.log
for w in "--workload c2" "--workload c3"; do
  tag=$(echo $w | awk '{print $2}')
  bash tools/ab_bench.sh ab10_$tag "$w" default corr16 corr8 > gpurun_out/ab10_$tag.txt 2>&1
done
