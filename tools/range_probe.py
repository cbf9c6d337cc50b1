"""One device batch inside a cudaProfilerStart/Stop range, for
`ncu --replay-mode app-range` (whole-range DRAM / L2 counters with the batch's
kernels running concurrently).  usage: range_probe.py <workload> <B> [opt=v,...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import _native  # noqa: E402

w, B = sys.argv[1], int(sys.argv[2])
opts = {}
if len(sys.argv) > 3:
    opts = {k: int(v) for k, v in (x.split("=") for x in sys.argv[3].split(","))}
gens = bench.workload_params(w)
dm = [torch.from_numpy(g()).cuda() for g, _ in gens]
sps = [sp for _, sp in gens]
ms = [dm[i % len(dm)] for i in range(B)]
ss = [sps[i % len(sps)] for i in range(B)]
s = torch.cuda.Stream()
with _native.thread_options(**opts):
    sc.calculate_coefficients_device_batch(ms, ss, stream=s)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    sc.calculate_coefficients_device_batch(ms, ss, stream=s)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
print("bytes of masks in the range:", sum(int(m.numel()) for m in ms))
