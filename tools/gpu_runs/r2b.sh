#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2b; mkdir -p $OUT
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-extras"
IFA_B200_WS=1 $B > $OUT/c2_ws_named.json 2>$OUT/err.txt
IFA_B200_WS=1 IFA_B200_LIB=build/ws_mb/libifa_b200.so $B > $OUT/c2_ws_mbar.json 2>>$OUT/err.txt
IFA_B200_WS=1 IFA_B200_LIB=build/ws_i2f/libifa_b200.so $B > $OUT/c2_ws_named_i2f.json 2>>$OUT/err.txt
$B > $OUT/c2_pp.json 2>>$OUT/err.txt
timeout 900 python -m pytest tests/test_gpu_dump.py tests/test_gpu_longseq.py -x -q --timeout 600 > $OUT/pytest_new.log 2>&1; echo "exit $?" >> $OUT/pytest_new.log
IFA_TEST_LOG=$PWD/$OUT/fast_log_pp.jsonl timeout 900 python -m pytest tests/test_gpu_parity.py -q -k fast > $OUT/pytest_fast_pp.log 2>&1; echo "exit $?" >> $OUT/pytest_fast_pp.log
IFA_B200_WS=1 IFA_TEST_LOG=$PWD/$OUT/fast_log_ws.jsonl timeout 900 python -m pytest tests/test_gpu_parity.py -q -k fast > $OUT/pytest_fast_ws.log 2>&1; echo "exit $?" >> $OUT/pytest_fast_ws.log
IFA_B200_WS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:int_flash -s 2 -c 1 \
  -o $OUT/ws_full python bench.py --steps 1 --warmup 3 --no-extras > $OUT/ncu_ws.log 2>&1
echo done > $OUT/DONE
