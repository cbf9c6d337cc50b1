set -u
mkdir -p gpurun_out
for w in ${@:-c2}; do
SC_OPTS=${SC_OPTS:-pack_tma=1,fused_bbox=1,grid_div=10} timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.sum,smsp__inst_executed.sum,launch__grid_size,sm__cycles_elapsed.avg.per_second --profile-from-start off --clock-control none --csv --log-file gpurun_out/cost_$w.csv python tools/batch_cost.py $w 4 > gpurun_out/cost_$w.log 2>&1
done
echo done
