#!/usr/bin/env bash
# One gpurun call: GPU tests, bench lines (C2 fast/exact, C3, C5), C4 MRE
# sweep, ncu launch list + full capture of the attention kernel.
#   gpurun --timeout 2400 -- 'bash tools/round_check.sh r1_v6'
set -u
TAG=${1:-check}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 300 python bench.py --no-extras --mode exact > $OUT/bench_c2_exact.json 2>> $OUT/bench.err
timeout 300 python bench.py --no-extras --workload c3 > $OUT/bench_c3.json 2>> $OUT/bench.err
timeout 600 python bench.py --no-extras --workload c5 > $OUT/bench_c5.json 2>> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_reference.json 2>> $OUT/bench.err
timeout 900 python tools/mre_sweep.py --out $OUT/c4_mre_sweep > $OUT/mre.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-extras > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:int_flash -s 2 -c 1 \
  -o $OUT/attn_full python bench.py --steps 1 --warmup 3 --no-extras > $OUT/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:pp_kernel<.int.128, .bool.0, .int.1" -s 2 -c 1 \
  -o $OUT/half_full python bench.py --steps 3 --warmup 3 > $OUT/ncu_half.log 2>&1
echo done > $OUT/DONE
