#!/usr/bin/env bash
# A/B timing of library variants on one box:
#   tools/ab_bench.sh TAG "bench args" lib1 lib2 ...   ("default" = in-tree build)
set -u
TAG=$1; ARGS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
for rep in 1 2; do
for L in "$@"; do
  if [ "$L" = default ]; then unset IFA_B200_LIB; else export IFA_B200_LIB=build/$L/libifa_b200.so; fi
  timeout 300 python bench.py --no-extras $ARGS > $OUT/$L.$rep.json 2>$OUT/$L.$rep.err
  python - "$OUT/$L.$rep.json" "$L" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
    print(sys.argv[2], "value", round(d["value"], 1), "attn_ms", round(d["breakdown_ms"]["attention"], 4))
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done
done
