#!/bin/bash
# One gpurun session: parity tests, smoke, bench, ncu launch list + full capture.
# usage (from this container): gpurun --timeout 1500 -- bash tools/gpu_check.sh [quick]
set -u
mkdir -p gpurun_out
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt 2>&1
timeout 600 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
if [ "${1:-}" != "quick" ]; then
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on \
      -k regex:"diam3d_pass1|pack_bits_v16|mc_cells|plane_pass1|boxes_extremes|scan_all|scatter_all|unit_filter|refine" -s 9 -c 9 \
      -o $OUT/prof -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_full.log 2>&1
fi
echo done
