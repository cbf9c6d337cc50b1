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
      --log-file $OUT/launches.csv python tools/one_roi.py > $OUT/ncu_bench.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on \
      -k regex:"pack_bits_v16|bits_bbox|mc_cells|scan_all|scatter_all|boxes_extremes|unit_filter|plane_boxes|plane_lb|plane_filter|diam_pass1|diam_refine" -s 12 -c 12 \
      -o $OUT/prof -f python tools/one_roi.py > $OUT/ncu_full.log 2>&1
fi
echo done
