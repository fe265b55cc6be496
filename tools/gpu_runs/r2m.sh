#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2m; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
echo done > $OUT/DONE
