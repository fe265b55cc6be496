#!/usr/bin/env bash
# One gpurun call: GPU tests + default bench line + ncu launch list.
set -u
TAG=${1:-quick}; shift || true
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests -m gpu -x -q "$@" > "$OUT/pytest_gpu.log" 2>&1
echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
timeout 600 python bench.py --no-extras > "$OUT/bench_c2.json" 2> "$OUT/bench_c2.err"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 3 --no-extras > "$OUT/ncu_launch.log" 2>&1
echo done > "$OUT/DONE"
