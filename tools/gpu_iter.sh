#!/bin/bash
# Iteration session: parity tests, stage marginals, bench lines (no CPU baseline).
set -u
mkdir -p gpurun_out
OUT=gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python tools/dbg_stages.py c2 c3 > $OUT/stages.log 2>&1
for w in ${WORKLOADS:-c2 c3}; do
  timeout 600 python bench.py --steps 20 --warmup 5 --workload $w --no-cpu-baseline > $OUT/bench_$w.json 2> $OUT/bench_$w.err
done
for extra in "$@"; do eval "$extra"; done
echo done
