#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2w; mkdir -p $OUT
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-extras"
$B > $OUT/c2_cur.json 2>>$OUT/err.txt
for v in kst3 vst3 g1d0 g1d2 poly8; do
IFA_B200_LIB=build/$v/libifa_b200.so $B > $OUT/c2_$v.json 2>>$OUT/err.txt
done
$B > $OUT/c2_cur2.json 2>>$OUT/err.txt
echo done > $OUT/DONE
