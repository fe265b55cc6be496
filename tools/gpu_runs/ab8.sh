set -u
mkdir -p gpurun_out/ab8
IFA_B200_LIB=build/corr/libifa_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dump.py tests/test_gpu_longseq.py tests/test_gpu_half.py tests/test_gpu_fp8.py tests/test_gpu_fuzz.py -q -x --timeout 300 > gpurun_out/ab8/pytest_corr.log 2>&1
for w in "--workload c2" "--workload c3" "--workload c5 --steps 3"; do
  tag=$(echo $w | awk '{print $2}')
  bash tools/ab_bench.sh ab8_$tag "$w" default corr > gpurun_out/ab8_$tag.txt 2>&1
done
