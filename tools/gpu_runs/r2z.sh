#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2z; mkdir -p $OUT
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-extras"
$B > $OUT/c2.json 2>>$OUT/err.txt
$B --workload c3 > $OUT/c3.json 2>>$OUT/err.txt
$B --workload c5 --steps 3 > $OUT/c5.json 2>>$OUT/err.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dump.py tests/test_gpu_half.py tests/test_gpu_fp8.py tests/test_gpu_longseq.py tests/test_gpu_fuzz.py -q -x --timeout 600 > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
echo done > $OUT/DONE
