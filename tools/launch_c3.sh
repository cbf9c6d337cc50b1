#!/bin/bash
# Per-kernel durations (+ instructions, L2/DRAM bytes) of one C3 ROI.
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/lc3.csv python tools/one_roi.py ${1:-c3} > gpurun_out/lc3.log 2>&1
