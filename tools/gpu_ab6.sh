set -u
mkdir -p gpurun_out
O=gpurun_out
SC_OPTS=pack_tma=1,fused_bbox=1 timeout 900 python tools/ab_batch.py pack_chain 0,1,2,4 c2 c4 c5 > $O/ab6_chain_tma.log 2>&1
SC_OPTS=pack_tma=0,fused_bbox=0 timeout 900 python tools/ab_batch.py pack_chain 0,1,2,4 c2 c4 > $O/ab6_chain_v16.log 2>&1
SC_OPTS=pack_tma=2,fused_bbox=1 timeout 900 python tools/ab_batch.py pack_chain 1,2 c2 c4 > $O/ab6_chain_tma2.log 2>&1
echo done
