#!/usr/bin/env bash
# round-2 first look: GPU tests, pipe rates, pp vs ws at C2
set -u
OUT=gpurun_out/r2a; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt
./tools/microbench/pipes > $OUT/pipes.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-extras > $OUT/c2_pp.json 2>$OUT/c2_pp.err
IFA_B200_WS=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-extras > $OUT/c2_ws.json 2>$OUT/c2_ws.err
IFA_B200_WS=1 IFA_WS_PINGPONG=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-extras > $OUT/c2_ws_nopp.json 2>$OUT/c2_ws_nopp.err
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
IFA_B200_WS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:int_flash -s 2 -c 1 \
  -o $OUT/ws_full python bench.py --steps 1 --warmup 3 --no-extras > $OUT/ncu_ws.log 2>&1
echo done > $OUT/DONE
