#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2s; mkdir -p $OUT
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-extras"
$B --mode exact > $OUT/c2_exact.json 2>>$OUT/err.txt
IFA_B200_LIB=build/base/libifa_b200.so $B --mode exact > $OUT/c2_exact_base.json 2>>$OUT/err.txt
IFA_B200_NO_PP=1 $B > $OUT/c2_quad.json 2>>$OUT/err.txt
IFA_B200_LIB=build/base/libifa_b200.so IFA_B200_NO_PP=1 $B > $OUT/c2_quad_base.json 2>>$OUT/err.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
echo done > $OUT/DONE
