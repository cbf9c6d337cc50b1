set -u
mkdir -p gpurun_out
O=gpurun_out
export SC_OPTS=pack_tma=1,slots=32,grid_div=10,fused_bbox=1
timeout 600 python tools/ab_batch.py pack_skip 1,0 c2 c4 c5 c3 > $O/ab5_skip.log 2>&1
timeout 600 python tools/nopack.py c2 c5 > $O/ab5_nopack.log 2>&1
echo done
