#!/bin/bash
# Parity tests + bench on every SURVEY workload (one GPU).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for w in c2 c5 c3 c4; do
  steps=30; [ $w = c3 ] && steps=5; [ $w = c4 ] && steps=300
  timeout 900 python bench.py --workload $w --steps $steps --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "$w rc=$?" >> gpurun_out/bench_$w.err
done

timeout 600 python bench.py --workload c3 --split --steps 5 --warmup 3 > gpurun_out/bench_c3_split.json 2> gpurun_out/bench_c3_split.err; echo "split rc=$?" >> gpurun_out/bench_c3_split.err
echo done
