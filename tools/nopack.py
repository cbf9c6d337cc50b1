"""Throughput of the post-pack pipeline alone: every slot first packs the
(same) mask once, then option pack_mode bit 2 skips the pack (the slot's bit
volume is reused, so results stay valid for a repeated mask).
usage: nopack.py w1 w2 ...  (SC_OPTS=k=v,... fixed options)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import _native  # noqa: E402

for kv in filter(None, os.environ.get("SC_OPTS", "").split(",")):
    k, v = kv.split("=")
    _native.set_option(k, int(v))
K = 200
for w in sys.argv[1:] or ["c2"]:
    rois, _ = bench.load_workload(w)
    m, sp = rois[0]
    d = torch.from_numpy(m).cuda()
    ref = sc.calculate_coefficients_device(d, sp).to_dict()
    for pm in (0, 4):
        _native.set_option("pack_mode", 0)
        sc.calculate_coefficients_device_batch([d] * 64, [sp] * 64)
        _native.set_option("pack_mode", pm)
        outs = sc.calculate_coefficients_device_batch([d] * 64, [sp] * 64)
        assert all(o.to_dict() == ref for o in outs)
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sc.calculate_coefficients_device_batch([d] * K, [sp] * K)
            torch.cuda.synchronize()
            best = min(best, (time.perf_counter() - t0) / K * 1e6)
        print(f"{w} pack_mode={pm}: {best:7.2f} us/ROI", flush=True)
    _native.set_option("pack_mode", 0)
