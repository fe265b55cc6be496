#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2ab; mkdir -p $OUT
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-extras"
for rep in 1 2; do
for w in c2 c3; do
$B --workload $w > $OUT/${w}_new_$rep.json 2>>$OUT/err.txt
IFA_B200_LIB=build/base3/libifa_b200.so $B --workload $w > $OUT/${w}_old_$rep.json 2>>$OUT/err.txt
done
done
$B --workload c5 --steps 3 > $OUT/c5_new.json 2>>$OUT/err.txt
IFA_B200_LIB=build/base3/libifa_b200.so $B --workload c5 --steps 3 > $OUT/c5_old.json 2>>$OUT/err.txt
echo done > $OUT/DONE
