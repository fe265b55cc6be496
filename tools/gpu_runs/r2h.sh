#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2h; mkdir -p $OUT
timeout 120 ./tools/microbench/sm_bw > $OUT/sm_bw.txt 2>&1
IFA_B200_STREAMED=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-extras > $OUT/c2_plain.json 2>>$OUT/err.txt
echo done > $OUT/DONE
