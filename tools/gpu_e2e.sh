#!/bin/bash
# GPU session: parity tests, host-scan probe, bench lines per workload.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
lscpu > $OUT/lscpu.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python tools/host_scan_probe.py > $OUT/host_probe.log 2>&1
for w in c2 c4 c5 c3; do
  timeout 600 python bench.py --steps 20 --warmup 5 --workload $w --no-cpu-baseline > $OUT/bench_$w.json 2> $OUT/bench_$w.err
done
echo done
