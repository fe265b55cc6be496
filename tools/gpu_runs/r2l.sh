#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2l; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_dump.py tests/test_multirank.py -q --timeout 800 > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-extras > $OUT/c2.json 2>>$OUT/err.txt
echo done > $OUT/DONE
