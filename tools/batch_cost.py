"""Workload for an ncu SM-time census of the batch path: a few ROIs through the
device batch entry with the batch options (grid_div etc.), after a warm-up.
usage: batch_cost.py <workload> [n_rois]  (SC_OPTS=k=v,... as in ab_batch.py)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import _native  # noqa: E402

for kv in filter(None, os.environ.get("SC_OPTS", "").split(",")):
    k, v = kv.split("=")
    _native.set_option(k, int(v))
w = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
rois, _ = bench.load_workload(w)
m, sp = rois[0]
d = torch.from_numpy(m).cuda()
_native.set_option("slots", 2)
sc.calculate_coefficients_device_batch([d] * 4, [sp] * 4)  # captures the slot graphs
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
sc.calculate_coefficients_device_batch([d] * n, [sp] * n)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
