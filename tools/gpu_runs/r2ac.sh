#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2ac; mkdir -p $OUT
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-extras"
for rep in 1 2; do
for w in c2 c3; do
$B --workload $w > $OUT/${w}_cur_$rep.json 2>>$OUT/err.txt
IFA_B200_LIB=build/pring/libifa_b200.so $B --workload $w > $OUT/${w}_ring_$rep.json 2>>$OUT/err.txt
done
done
IFA_B200_LIB=build/pring/libifa_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dump.py tests/test_gpu_half.py tests/test_gpu_fp8.py -q -x --timeout 600 > $OUT/pytest_ring.log 2>&1; echo "exit $?" >> $OUT/pytest_ring.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dump.py -q -x -k "fast or dump" --timeout 600 > $OUT/pytest_cur.log 2>&1; echo "exit $?" >> $OUT/pytest_cur.log
echo done > $OUT/DONE
