#!/usr/bin/env bash
set -u
OUT=gpurun_out/r2f; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 600 python bench.py --workload c3 --no-extras > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 900 python -m pytest tests/test_multirank.py -x -q --timeout 800 > $OUT/pytest_multirank.log 2>&1; echo "exit $?" >> $OUT/pytest_multirank.log
echo done > $OUT/DONE
