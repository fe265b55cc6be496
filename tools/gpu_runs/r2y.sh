#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2y; mkdir -p $OUT
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-extras"
for rep in 1 2; do
$B > $OUT/c2_cur_$rep.json 2>>$OUT/err.txt
IFA_B200_LIB=build/mcvt/libifa_b200.so $B > $OUT/c2_mcvt_$rep.json 2>>$OUT/err.txt
done
IFA_B200_LIB=build/mcvt/libifa_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dump.py -q -x -k "fast or dump" --timeout 300 > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
echo done > $OUT/DONE
