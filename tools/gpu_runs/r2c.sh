#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2c; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_host_pipeline.py tests/test_gpu_dump.py -x -q --timeout 600 > $OUT/pytest_new.log 2>&1; echo "exit $?" >> $OUT/pytest_new.log
IFA_B200_WS=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -k fast > $OUT/pytest_fast_ws.log 2>&1; echo "exit $?" >> $OUT/pytest_fast_ws.log
timeout 300 ./oracle/_ref/verify_gpu > $OUT/verify_gpu.log 2>&1; echo "exit $?" >> $OUT/verify_gpu.log
for pp in 1 0; do
IFA_B200_WS=1 IFA_WS_PINGPONG=$pp IFA_B200_LIB=build/trace/libifa_b200.so timeout 300 python tools/ws_trace.py 128 4096 60 > $OUT/trace_pp$pp.txt 2>&1
done
IFA_B200_WS=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-extras > $OUT/c2_ws.json 2>$OUT/err.txt
echo done > $OUT/DONE
