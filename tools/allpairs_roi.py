"""C2 with pruning disabled (every pair through pass 1): for ncu captures of
the brute-force pass-1 roofline."""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_2510_02894_b200 as sc
from paper_2510_02894_b200 import _native

rois, _ = bench.load_workload(sys.argv[1] if len(sys.argv) > 1 else "c2")
mask, sp = rois[0]
d = torch.from_numpy(mask).cuda()
_native.set_option("prune", 0)
for _ in range(2):
    c = sc.calculate_coefficients_device(d, sp)
torch.cuda.synchronize()
print(c.to_dict())
