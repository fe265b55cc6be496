#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2k; mkdir -p $OUT
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-extras"
IFA_B200_WS=1 $B > $OUT/c2_ws_sp.json 2>>$OUT/err.txt
IFA_B200_WS=1 $B --dist uniform > $OUT/c2u_ws_sp.json 2>>$OUT/err.txt
IFA_B200_WS=1 IFA_B200_LIB=build/ws_sp0/libifa_b200.so $B > $OUT/c2_ws_sp0.json 2>>$OUT/err.txt
$B > $OUT/c2_pp.json 2>>$OUT/err.txt
IFA_B200_WS=1 $B --workload c3 > $OUT/c3_ws_sp.json 2>>$OUT/err.txt
IFA_B200_WS=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dump.py tests/test_gpu_longseq.py -q -k "fast or dump or tiles" --timeout 600 > $OUT/pytest_ws.log 2>&1; echo "exit $?" >> $OUT/pytest_ws.log
echo done > $OUT/DONE
