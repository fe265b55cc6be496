#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2x; mkdir -p $OUT
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-extras"
$B > $OUT/c2_cur.json 2>>$OUT/err.txt
$B --dist uniform > $OUT/c2u_cur.json 2>>$OUT/err.txt
for v in sp1 sp32b; do
IFA_B200_LIB=build/$v/libifa_b200.so $B > $OUT/c2_$v.json 2>>$OUT/err.txt
IFA_B200_LIB=build/$v/libifa_b200.so $B --dist uniform > $OUT/c2u_$v.json 2>>$OUT/err.txt
done
echo done > $OUT/DONE
