set -u
mkdir -p gpurun_out/ab9
export IFA_B200_LIB=build/corr/libifa_b200.so
timeout 180 python -m pytest "tests/test_gpu_parity.py::test_fast_mode_within_tolerance" -q -x --timeout 60 > gpurun_out/ab9/pytest_quick.log 2>&1
echo "rc $?" >> gpurun_out/ab9/pytest_quick.log
timeout 120 python bench.py --no-extras --workload c2 > gpurun_out/ab9/c2.json 2> gpurun_out/ab9/c2.err
echo "rc $?" >> gpurun_out/ab9/c2.err
