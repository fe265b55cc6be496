#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2ae; mkdir -p $OUT
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-extras"
for rep in 1 2; do
for w in c2 c3; do
$B --workload $w > $OUT/${w}_cur_$rep.json 2>>$OUT/err.txt
IFA_B200_LIB=build/r104/libifa_b200.so $B --workload $w > $OUT/${w}_r104_$rep.json 2>>$OUT/err.txt
done
done
echo done > $OUT/DONE
