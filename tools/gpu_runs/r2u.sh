#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2u; mkdir -p $OUT
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-extras"
for rep in 1 2 3; do
$B > $OUT/c2_cur_$rep.json 2>>$OUT/err.txt
IFA_B200_LIB=build/base/libifa_b200.so $B > $OUT/c2_base_$rep.json 2>>$OUT/err.txt
done
echo done > $OUT/DONE
