#!/bin/bash
# Quick GPU session: parity tests + bench variants (no ncu).
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
SC_PASS1=scalar timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_scalar.json 2>> gpurun_out/bench.err
for extra in "$@"; do eval "$extra"; done
echo done
