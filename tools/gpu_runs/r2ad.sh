#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2ad; mkdir -p $OUT
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-extras"
for rep in 1 2; do
$B > $OUT/c2_new_$rep.json 2>>$OUT/err.txt
IFA_B200_LIB=build/base3/libifa_b200.so $B > $OUT/c2_old_$rep.json 2>>$OUT/err.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_runtime.py tests/test_gpu_step.py -q -x --timeout 600 > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
echo done > $OUT/DONE
