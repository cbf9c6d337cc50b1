"""Marginal batch cost of each pipeline stage for the batch configuration
(TMA pack with fused bbox): throughput with only the first N kernels enqueued
per ROI (option debug_stages; results invalid, timing only).  Distinct masks
cycle as in the bench.  usage: stage_marginals_batch.py workload [K]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import _native  # noqa: E402

NAMES = ["init", "pack+bbox", "mc_cells", "scan_all", "scatter_all", "boxes_extremes",
         "unit_filter+expand", "plane_boxes", "plane_lb", "plane_filter", "pass1", "refine"]
w = sys.argv[1] if len(sys.argv) > 1 else "c2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 200
gens = bench.workload_params(w)[:64]
dm = [torch.from_numpy(g()).cuda() for g, _ in gens]
sps = [sp for _, sp in gens]
ms = [dm[i % len(dm)] for i in range(K)]
ss = [sps[i % len(sps)] for i in range(K)]
def run():
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sc.calculate_coefficients_device_batch(ms, ss)
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) / K * 1e6)
    return best


sc.calculate_coefficients_device_batch(ms[:64], ss[:64])
full = run()
print(f"{w} full pipeline (planar chain forked) {full:7.2f} us/ROI", flush=True)
# Descending cuts; a cut before scatter_all leaves the self-cleaning sort
# histograms dirty, so those come last and nothing valid runs after them.
res = {}
for n in (12, 11, 10, 9, 8, 7, 6, 5, 3, 2):
    _native.set_option("debug_stages", n)
    try:
        sc.calculate_coefficients_device_batch(ms[:64], ss[:64])
        res[n] = run()
    except Exception as exc:  # results of cut pipelines are invalid (EmptyRoi etc.)
        print(f"stages<={n}: {exc}", flush=True)
        break
prev = 0.0
for n in sorted(res):
    print(f"{w} stages<={n:2d} (+{NAMES[n - 1]:18s}) {res[n]:7.2f} us/ROI  marginal "
          f"{res[n] - prev:+6.2f}", flush=True)
    prev = res[n]
