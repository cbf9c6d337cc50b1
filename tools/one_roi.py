"""A few single-ROI calls for ncu captures: no probes, no batch overlap.

usage: python tools/one_roi.py [c2|c3|c5]   (default c2)"""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_2510_02894_b200 as sc

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
rois, _ = bench.load_workload(name)
mask, sp = rois[0]
d = torch.from_numpy(mask).cuda()
for _ in range(3):
    c = sc.calculate_coefficients_device(d, sp)
torch.cuda.synchronize()
print(c.to_dict())
