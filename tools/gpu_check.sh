#!/usr/bin/env bash
# One gpurun call: GPU parity tests, smoke, bench lines, ncu launch list and
# one `ncu --set full` capture of the attention kernel.  Every step has its
# own timeout so a hang cannot eat the whole call.
#   gpurun --timeout 1800 -- 'bash tools/gpu_check.sh [tag]'
set -u
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
echo "smoke exit $?" >> "$OUT/smoke.log"
timeout 600 python bench.py > "$OUT/bench_c2.json" 2> "$OUT/bench_c2.err"
timeout 300 python bench.py --dist uniform --no-extras > "$OUT/bench_c2_uniform.json" 2> "$OUT/bench_c2_uniform.err"
timeout 300 python bench.py --workload c3 --no-extras > "$OUT/bench_c3.json" 2> "$OUT/bench_c3.err"
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-extras > "$OUT/ncu_launch.log" 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:int_flash -s 2 -c 1 \
    -o "$OUT/attn_full" python bench.py --steps 1 --warmup 3 --no-extras > "$OUT/ncu_full.log" 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:quantize_rows -s 4 -c 1 \
    -o "$OUT/quant_full" python bench.py --steps 1 --warmup 3 --no-extras > "$OUT/ncu_quant.log" 2>&1
fi
echo done > "$OUT/DONE"
