#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2j; mkdir -p $OUT
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-extras"
for v in default sp0 sp8 sp32; do
  if [ $v = default ]; then L=""; else L="IFA_B200_LIB=build/$v/libifa_b200.so"; fi
  env $L $B > $OUT/c2_$v.json 2>>$OUT/err.txt
  env $L $B --dist uniform > $OUT/c2u_$v.json 2>>$OUT/err.txt
done
$B --workload c3 > $OUT/c3_default.json 2>>$OUT/err.txt
IFA_B200_LIB=build/sp0/libifa_b200.so $B --workload c3 > $OUT/c3_sp0.json 2>>$OUT/err.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dump.py tests/test_gpu_longseq.py tests/test_gpu_fuzz.py -q --timeout 600 > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
echo done > $OUT/DONE
