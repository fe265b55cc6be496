#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2aa; mkdir -p $OUT
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-extras"
for rep in 1 2; do
$B --workload c3 > $OUT/c3_new_$rep.json 2>>$OUT/err.txt
IFA_B200_LIB=build/base2/libifa_b200.so $B --workload c3 > $OUT/c3_old_$rep.json 2>>$OUT/err.txt
$B > $OUT/c2_new_$rep.json 2>>$OUT/err.txt
IFA_B200_LIB=build/base2/libifa_b200.so $B > $OUT/c2_old_$rep.json 2>>$OUT/err.txt
done
echo done > $OUT/DONE
