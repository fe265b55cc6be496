#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2e; mkdir -p $OUT
L=build/ws_cp/libifa_b200.so
IFA_B200_WS=1 IFA_B200_LIB=$L timeout 600 python -m pytest tests/test_gpu_dump.py -x -q > $OUT/pytest_dump_cp.log 2>&1; echo "exit $?" >> $OUT/pytest_dump_cp.log
IFA_B200_WS=1 IFA_B200_LIB=$L timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k fast > $OUT/pytest_fast_cp.log 2>&1; echo "exit $?" >> $OUT/pytest_fast_cp.log
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-extras"
IFA_B200_WS=1 IFA_B200_LIB=$L $B > $OUT/c2_ws_cp.json 2>$OUT/err.txt
IFA_B200_WS=1 $B > $OUT/c2_ws.json 2>>$OUT/err.txt
IFA_B200_WS=1 IFA_B200_LIB=build/ws_cp_trace/libifa_b200.so timeout 300 python tools/ws_trace.py 128 4096 60 > $OUT/trace_cp.txt 2>&1
echo done > $OUT/DONE
