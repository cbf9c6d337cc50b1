set -u
mkdir -p gpurun_out
O=gpurun_out
SC_OPTS=pack_tma=1 timeout 600 python tools/ab_batch.py slots 16,24,32,12 c2 c4 > $O/ab_slots_tma1.log 2>&1
SC_OPTS=pack_tma=0 timeout 600 python tools/ab_batch.py slots 16,24,32 c2 > $O/ab_slots_tma0.log 2>&1
SC_OPTS=pack_tma=1 timeout 600 python tools/ab_batch.py grid_div 5,3,8,12 c2 c5 > $O/ab_griddiv_tma1.log 2>&1
SC_OPTS=pack_tma=1 timeout 600 python tools/ab_batch.py pack_mode 0,4 c2 > $O/ab_nopack.log 2>&1 || true
echo done
