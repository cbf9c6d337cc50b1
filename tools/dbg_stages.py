"""Marginal batch cost of each pipeline stage: throughput with only the first N
kernels enqueued per ROI (option debug_stages; results invalid, timing only)."""
import sys, time
sys.path.insert(0, '.')
import torch, bench
import paper_2510_02894_b200 as sc
from paper_2510_02894_b200 import _native

NAMES = ["init", "pack", "bbox", "mc", "scan_all", "scatter", "boxes",
         "unit_filter", "plane_boxes", "plane_lb", "plane_filter", "pass1", "refine"]
for w in sys.argv[1:] or ["c2"]:
    rois, _ = bench.load_workload(w)
    m, sp = rois[0]
    d = torch.from_numpy(m).cuda()
    # Descending, full pipeline first: runs cut before scatter_all leave the
    # self-cleaning histograms dirty, so they go last (and only once per process).
    res = {}
    for n in (13, 12, 11, 10, 9, 8, 7, 6) + ((4, 3) if w == sys.argv[-1] else ()):
        _native.set_option("debug_stages", n)
        sc.calculate_coefficients_device_batch([d] * 16, [sp] * 16)
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            sc.calculate_coefficients_device_batch([d] * 100, [sp] * 100)
            torch.cuda.synchronize(); best = min(best, (time.perf_counter() - t0) / 100 * 1e6)
        res[n] = best
    _native.set_option("debug_stages", 0)
    prev = 0.0
    for n in sorted(res):
        print(f"{w} stages<={n:2d} (+{NAMES[n-1]:15s}) {res[n]:7.1f} us/ROI  marginal {res[n] - prev:+6.1f}", flush=True)
        prev = res[n]
