#!/bin/bash
# Full ncu capture of selected kernels of one single-ROI call.
# usage: gpu_ncu.sh <workload> <kernel-regex> <tag>
set -u
mkdir -p gpurun_out
w=${1:-c3}; re=${2:-mc_cells}; tag=${3:-$w}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$re" -s ${4:-0} -c ${5:-8} \
    -o gpurun_out/prof_$tag -f python tools/one_roi.py $w > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full_$tag.log
