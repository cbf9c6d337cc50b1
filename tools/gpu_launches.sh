#!/bin/bash
# Per-kernel launch list (cold, serialised) of a few single-ROI calls per workload.
set -u
mkdir -p gpurun_out
for w in ${@:-c2 c3}; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$w.csv python tools/one_roi.py $w > gpurun_out/ncu_$w.log 2>&1
done
echo done
