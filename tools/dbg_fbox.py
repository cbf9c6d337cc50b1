"""Pack with fused bbox vs pack + bits_bbox: per-stage times and batch throughput."""
import sys, time
sys.path.insert(0, '.')
import torch
import bench
import paper_2510_02894_b200 as sc
from paper_2510_02894_b200 import _native
_native.set_option("stage_times", 2)  # per-stage events for last_kernel_times

for w in ("c2", "c3", "c5"):
    rois, _ = bench.load_workload(w)
    m, sp = rois[0]
    d = torch.from_numpy(m).cuda()
    for fb in (1, 0):
        _native.set_option("fused_bbox", fb)
        ref = None
        ts = []
        for _ in range(10):
            c = sc.calculate_coefficients_device(d, sp)
            ts.append(_native.last_kernel_times(0))
            ref = ref or c.to_dict()
            assert c.to_dict() == ref
        pk = sorted(t["pack_ms"] for t in ts)[5] * 1e3
        mc = sorted(t["mc_ms"] for t in ts)[5] * 1e3
        sc.calculate_coefficients_device_batch([d] * 16, [sp] * 16)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sc.calculate_coefficients_device_batch([d] * 100, [sp] * 100)
        torch.cuda.synchronize()
        print(w, "fused_bbox", fb, f"pack {pk:.1f} us  mc {mc:.1f} us  batch {100 / (time.perf_counter() - t0):.0f} ROIs/s", flush=True)
