set -u
OUT=gpurun_out/r1_fast1; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
for m in exact fast; do
  timeout 300 python bench.py --no-extras --mode $m > $OUT/bench_c2_$m.json 2>$OUT/bench_c2_$m.err
  timeout 300 python bench.py --no-extras --mode $m --dist uniform > $OUT/bench_c2u_$m.json 2>$OUT/bench_c2u_$m.err
  timeout 300 python bench.py --no-extras --mode $m --workload c3 > $OUT/bench_c3_$m.json 2>$OUT/bench_c3_$m.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:int_flash -s 2 -c 1 -o $OUT/attn_fast python bench.py --steps 1 --warmup 3 --no-extras --mode fast > $OUT/ncu_full.log 2>&1
