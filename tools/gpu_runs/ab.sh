#!/usr/bin/env bash
# A/B of library builds on the same box: bench lines per workload, the
# libraries interleaved, two rounds.  usage: ab.sh TAG "c2 c5" lib1 lib2 ...
set -u
TAG=$1; W=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
for rep in 1 2; do
  for w in $W; do
    for lib in "$@"; do
      st=""; [ "$w" = c5 ] && st="--steps 3"
      IFA_B200_LIB=$lib timeout 600 python bench.py --no-extras --workload $w $st > $OUT/${w}_$(basename $(dirname $lib))_$rep.json 2>> $OUT/err.log
    done
  done
done
echo done > $OUT/DONE
