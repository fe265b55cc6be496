#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2d; mkdir -p $OUT
./tools/microbench/code_loop > $OUT/code_loop.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
echo done > $OUT/DONE
