#!/usr/bin/env bash
# Round-2 check: GPU tests, smoke, bench lines (C2 with extras, C2 exact, C3,
# C5, C1), NO_PP A/B (kind::i8 P.V quad kernel), reference arm, ncu launch
# list + full captures of the attention and quantize kernels.
set -u
TAG=${1:-r2_check}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "exit $?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 300 python bench.py --no-extras --mode exact > $OUT/bench_c2_exact.json 2>> $OUT/bench.err
timeout 600 python bench.py --no-extras --workload c3 > $OUT/bench_c3.json 2>> $OUT/bench.err
timeout 900 python bench.py --no-extras --workload c5 --steps 5 > $OUT/bench_c5.json 2>> $OUT/bench.err
timeout 300 python bench.py --no-extras --workload c1 > $OUT/bench_c1.json 2>> $OUT/bench.err
for w in c2 c3; do IFA_B200_NO_PP=1 timeout 600 python bench.py --no-extras --workload $w > $OUT/bench_${w}_i8pv.json 2>> $OUT/bench.err; done
IFA_B200_NO_PP=1 timeout 900 python bench.py --no-extras --workload c5 --steps 3 > $OUT/bench_c5_i8pv.json 2>> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_reference.json 2>> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-extras > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:int_flash -s 2 -c 1 \
  -o $OUT/attn_full python bench.py --steps 1 --warmup 3 --no-extras > $OUT/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:slice_quantize_fused -s 2 -c 1 \
  -o $OUT/quant_v_full python bench.py --steps 1 --warmup 3 --no-extras > $OUT/ncu_quant.log 2>&1
echo done > $OUT/DONE
