"""Throughput of the post-pack pipeline alone: after every slot has packed the
(same) mask once, option pack_mode bit 2 skips the pack (the slot's bit volume
is reused, so results stay valid for a repeated mask)."""
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import _native  # noqa: E402

for w in sys.argv[1:] or ["c2"]:
    rois, _ = bench.load_workload(w)
    m, sp = rois[0]
    d = torch.from_numpy(m).cuda()
    ref = sc.calculate_coefficients_device(d, sp).to_dict()
    for pm, slots in ((0, 8), (4, 8), (4, 4), (4, 2), (4, 1), (0, 1)):
        _native.set_option("slots", slots)
        _native.set_option("pack_mode", 0)
        sc.calculate_coefficients_device_batch([d] * 16, [sp] * 16)
        _native.set_option("pack_mode", pm)
        outs = sc.calculate_coefficients_device_batch([d] * 16, [sp] * 16)
        assert all(o.to_dict() == ref for o in outs)
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sc.calculate_coefficients_device_batch([d] * 100, [sp] * 100)
            torch.cuda.synchronize()
            best = min(best, (time.perf_counter() - t0) / 100 * 1e6)
        print(f"{w} pack_mode {pm} slots {slots}: {best:6.1f} us/ROI", flush=True)
    _native.set_option("pack_mode", 0)
    _native.set_option("slots", 8)
