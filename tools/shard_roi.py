"""Shard-entry calls for ncu launch lists: the one-call pair-grid shard entry
(shard 0 of N) and the two-phase slab split (all N shards simulated).

usage: python tools/shard_roi.py [c2|c3] [N] [pairs|slab]"""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_2510_02894_b200 as sc
from paper_2510_02894_b200 import sharding

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mode = sys.argv[3] if len(sys.argv) > 3 else "pairs"
g, sp = bench.workload_params(name)[0]
d = torch.from_numpy(g()).cuda()
sq = torch.zeros(4, dtype=torch.float64, device="cuda")
for _ in range(2):
    if mode == "pairs":
        c = sc.calculate_coefficients_shard(d, sp, 0, n, sq)
    else:
        c = sharding.simulate_slab_shards(d, sp, n)
torch.cuda.synchronize()
print(c if isinstance(c, dict) else c.to_dict())
