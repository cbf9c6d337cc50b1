set -u
mkdir -p gpurun_out
O=gpurun_out
SC_OPTS=pack_tma=1,slots=32 timeout 600 python tools/ab_batch.py fused_bbox 0,1 c2 c4 c5 c3 > $O/ab_fbox.log 2>&1
SC_OPTS=pack_tma=1,slots=32,fused_bbox=1 timeout 600 python tools/ab_batch.py grid_div 5,6,8,10,14 c2 c5 c3 > $O/ab_griddiv2.log 2>&1
SC_OPTS=pack_tma=1,slots=32,fused_bbox=1 timeout 600 python tools/ab_batch.py pack_mode 0,2 c2 c5 > $O/ab_lowprio.log 2>&1
SC_OPTS=slots=32,fused_bbox=1 timeout 600 python tools/ab_batch.py pack_tma 1,2,3 c2 c3 > $O/ab_tma_fbox.log 2>&1
echo done
