"""Batch throughput (device-resident, pipelined) vs option pack_mode and the
number of pipeline stages enqueued (debug_stages; cut runs are timing only)."""
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import _native  # noqa: E402


def rate(d, sp, n=100):
    sc.calculate_coefficients_device_batch([d] * 16, [sp] * 16)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sc.calculate_coefficients_device_batch([d] * n, [sp] * n)
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) / n * 1e6)
    return best


for w in sys.argv[1:] or ["c2"]:
    rois, _ = bench.load_workload(w)
    m, sp = rois[0]
    d = torch.from_numpy(m).cuda()
    ref = sc.calculate_coefficients_device(d, sp).to_dict()
    for pm in ((0, 1, 2, 3) if w == (sys.argv[1:] or ["c2"])[-1] else (1, 2, 3, 0)):
        _native.set_option("pack_mode", pm)
        assert sc.calculate_coefficients_device(d, sp).to_dict() == ref, pm
        line = []
        # cuts before scatter_all leave the self-cleaning histograms dirty: only
        # on the last workload, after every full run
        for n in (14, 7) + ((4, 3) if w == (sys.argv[1:] or ["c2"])[-1] else ()):
            _native.set_option("debug_stages", n)
            line.append(f"<= {n:2d}: {rate(d, sp):6.1f}")
        _native.set_option("debug_stages", 0)
        print(f"{w} pack_mode {pm}: us/ROI " + "  ".join(line), flush=True)
    _native.set_option("pack_mode", 0)
