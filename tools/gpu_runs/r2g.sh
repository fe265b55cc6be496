#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2g; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_step.py -x -q --timeout 300 > $OUT/pytest_step.log 2>&1; echo "exit $?" >> $OUT/pytest_step.log
for s in 8 12 16 20; do
IFA_B200_QUANT_SMS=$s timeout 300 python bench.py --steps 10 --warmup 3 --no-extras > $OUT/c2_q$s.json 2>>$OUT/err.txt
done
IFA_B200_STREAMED=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-extras > $OUT/c2_plain.json 2>>$OUT/err.txt
timeout 300 python bench.py --workload c5 --steps 3 --warmup 3 --no-extras > $OUT/c5.json 2>>$OUT/err.txt
IFA_B200_STREAMED=0 timeout 300 python bench.py --workload c5 --steps 3 --warmup 3 --no-extras > $OUT/c5_plain.json 2>>$OUT/err.txt
timeout 900 python -m pytest tests/test_multirank.py -x -q --timeout 800 > $OUT/pytest_multirank.log 2>&1; echo "exit $?" >> $OUT/pytest_multirank.log
echo done > $OUT/DONE
