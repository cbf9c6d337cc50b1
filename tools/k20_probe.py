"""Device-batch time of K ROIs (the bench's timed region) vs slot count.

usage: python tools/k20_probe.py [K] [workload] [clocks] [warmk]"""
import os
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import _native  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
SLOTS = (16,) if "only16" in sys.argv[3:] else tuple(int(x) for x in os.environ.get("SLOTS", "12,16").split(","))
w = sys.argv[2] if len(sys.argv) > 2 else "c2"
clocks = "clocks" in sys.argv[3:]
warm_k = "warmk" in sys.argv[3:]  # NVML sampler running, as in bench.py
for kv in filter(None, os.environ.get("SC_OPTS", "").split(",")):  # fixed extra options
    k, v = kv.split("=")
    _native.set_option(k, int(v))
rois, _ = bench.load_workload(w)
d = [torch.from_numpy(m).cuda() for m, _ in rois]
sps = [sp for _, sp in rois]
s = torch.cuda.Stream()
for slots in SLOTS:
    _native.set_option("slots", slots)
    sc.calculate_coefficients_device_batch([d[i % len(d)] for i in range(32)],
                                           [sps[i % len(d)] for i in range(32)], stream=s)
    if warm_k:  # a second warm-up batch of exactly K ROIs
        sc.calculate_coefficients_device_batch([d[i % len(d)] for i in range(K)],
                                               [sps[i % len(d)] for i in range(K)], stream=s)
    best = []
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cs = bench.ClockSampler(torch.cuda.current_device()) if clocks else None
        if cs:
            cs.__enter__()
        e0.record(s)
        sc.calculate_coefficients_device_batch([d[i % len(d)] for i in range(K)],
                                               [sps[i % len(d)] for i in range(K)], stream=s)
        e1.record(s)
        torch.cuda.synchronize()
        if cs:
            cs.__exit__(None, None, None)
        best.append(e0.elapsed_time(e1))
    runs = list(best)
    best.sort()
    print(f"{w} K={K} slots={slots}: median {best[2] * 1e3 / K:.1f} us/ROI "
          f"({K / best[2] * 1e3:.0f} ROIs/s), best {best[0] * 1e3 / K:.1f}, runs {[round(b * 1e3 / K, 1) for b in runs]}")
