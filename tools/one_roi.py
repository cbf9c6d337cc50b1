"""A few single-ROI calls for ncu captures: no probes, no batch overlap.

usage: python tools/one_roi.py [c2|c3|c5] [tma]   (default c2; "tma": the
batch path's TMA pack with the fused bbox instead of the 128-bit-load pack)"""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_2510_02894_b200 as sc
from paper_2510_02894_b200 import _native

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
opts = {"pack_tma_single": 1, "fused_bbox_single": 1} if "tma" in sys.argv[2:] else {}
g, sp = bench.workload_params(name)[0]  # the workload's first ROI only
mask = g()
d = torch.from_numpy(mask).cuda()
with _native.thread_options(**opts):
    for _ in range(3):
        c = sc.calculate_coefficients_device(d, sp)
torch.cuda.synchronize()
print(c.to_dict())
