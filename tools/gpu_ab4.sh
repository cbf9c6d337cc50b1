set -u
mkdir -p gpurun_out
O=gpurun_out
export AB_NOCHECK=1
SC_OPTS=debug_stages=1,slots=32 timeout 600 python tools/ab_batch.py debug_empty 0,4,8,16,32 c2 > $O/ab_empty.log 2>&1
SC_OPTS=debug_stages=1,slots=16 timeout 600 python tools/ab_batch.py debug_empty 0,8,16 c2 >> $O/ab_empty.log 2>&1
SC_OPTS=pack_mode=4,pack_tma=1,fused_bbox=1,grid_div=10 timeout 600 python tools/ab_batch.py slots 8,16,32 c2 > $O/ab_nopack_slots.log 2>&1
SC_OPTS=pack_mode=4,pack_tma=1,fused_bbox=1,slots=32 timeout 600 python tools/ab_batch.py grid_div 5,10,20 c2 >> $O/ab_nopack_slots.log 2>&1
SC_OPTS=pack_mode=4,pack_tma=1,fused_bbox=1,slots=32,grid_div=10 timeout 600 python tools/ab_batch.py fork 1,0 c2 >> $O/ab_nopack_slots.log 2>&1
echo done
