#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2v; mkdir -p $OUT
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-extras"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dump.py tests/test_gpu_half.py tests/test_gpu_fp8.py tests/test_gpu_longseq.py tests/test_gpu_fuzz.py -q -x --timeout 600 > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for rep in 1 2; do
$B > $OUT/c2_tma_$rep.json 2>>$OUT/err.txt
IFA_B200_NO_OTMA=1 $B > $OUT/c2_notma_$rep.json 2>>$OUT/err.txt
done
$B --workload c3 > $OUT/c3_tma.json 2>>$OUT/err.txt
IFA_B200_NO_OTMA=1 $B --workload c3 > $OUT/c3_notma.json 2>>$OUT/err.txt
echo done > $OUT/DONE
