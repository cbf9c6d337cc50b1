"""Latency of one synchronous call per ROI (device mask), with and without the
per-stage event nodes, and the C-level time share (wall per call)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import _native  # noqa: E402

for w in sys.argv[1:] or ["c2"]:
    rois, _ = bench.load_workload(w)
    m, sp = rois[0]
    d = torch.from_numpy(m).cuda()
    for st in (2, 1, 0):
        _native.set_option("stage_times", st)
        for _ in range(10):
            sc.calculate_coefficients_device(d, sp)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(200):
            sc.calculate_coefficients_device(d, sp)
        dt = (time.perf_counter() - t0) / 200 * 1e6
        print(f"{w} stage_times={st}: {dt:.1f} us per synchronous call", flush=True)
    _native.set_option("stage_times", 0)
