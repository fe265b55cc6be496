#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2p; mkdir -p $OUT
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-extras"
for rep in 1 2; do
$B > $OUT/c2_ring0_$rep.json 2>>$OUT/err.txt
IFA_B200_LIB=build/hw1/libifa_b200.so $B > $OUT/c2_ring1_$rep.json 2>>$OUT/err.txt
IFA_B200_LIB=build/base/libifa_b200.so $B > $OUT/c2_base_$rep.json 2>>$OUT/err.txt
done
echo done > $OUT/DONE
