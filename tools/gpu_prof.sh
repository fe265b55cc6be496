#!/usr/bin/env bash
# One gpurun call: bench line + ncu --set full of the attention kernel only.
#   gpurun --timeout 900 -- 'bash tools/gpu_prof.sh tag [bench args]'
set -u
TAG=${1:-prof}; shift || true
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 300 python bench.py --no-extras "$@" > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:int_flash -s 2 -c 1 \
  -o "$OUT/attn_full" python bench.py --steps 1 --warmup 3 --no-extras "$@" > "$OUT/ncu_full.log" 2>&1
echo done > "$OUT/DONE"
