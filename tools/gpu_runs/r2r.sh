#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2r; mkdir -p $OUT
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-extras"
IFA_B200_WS=1 $B > $OUT/c2_ws.json 2>>$OUT/err.txt
IFA_B200_WS=1 IFA_WS_PINGPONG=0 $B > $OUT/c2_ws_nopp.json 2>>$OUT/err.txt
$B > $OUT/c2_pp.json 2>>$OUT/err.txt
IFA_B200_WS=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dump.py -q -x -k "fast or dump" --timeout 600 > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
echo done > $OUT/DONE
