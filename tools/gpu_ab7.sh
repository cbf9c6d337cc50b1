set -u
mkdir -p gpurun_out
O=gpurun_out
SC_OPTS=pack_tma=1,fused_bbox=1 timeout 900 python tools/ab_batch.py pack_chain 3,4,5,6,8,12 c2 c4 c5 > $O/ab7_chain.log 2>&1
SC_OPTS=pack_tma=1,fused_bbox=1,pack_chain=5 timeout 900 python tools/ab_batch.py grid_div 6,10,16 c2 c4 > $O/ab7_gd.log 2>&1
echo done
