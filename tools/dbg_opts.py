"""Batch throughput (device-resident, pipelined) per workload vs one option's
values; results must not change.  usage: dbg_opts.py OPTION v1,v2,.. w1 w2 .."""
import os
import sys
import time

sys.path.insert(0, '.')
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import _native  # noqa: E402


def rate(d, sp, n=100, ref=None):
    outs = sc.calculate_coefficients_device_batch([d] * 16, [sp] * 16)
    if ref is not None:
        assert all(o.to_dict() == ref for o in outs), "batch result differs"

    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sc.calculate_coefficients_device_batch([d] * n, [sp] * n)
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) / n * 1e6)
    return best


opt, vals = sys.argv[1], [int(v) for v in sys.argv[2].split(",")]
for kv in filter(None, os.environ.get("SC_OPTS", "").split(",")):  # fixed extra options
    k, v = kv.split("=")
    _native.set_option(k, int(v))
for w in sys.argv[3:]:
    rois, _ = bench.load_workload(w)
    m, sp = rois[0]
    d = torch.from_numpy(m).cuda()
    ref = sc.calculate_coefficients_device(d, sp).to_dict()
    for v in vals:
        _native.set_option(opt, v)
        assert sc.calculate_coefficients_device(d, sp).to_dict() == ref, (opt, v)
        one = []
        _native.set_option("stage_times", 2)
        for _ in range(10):
            sc.calculate_coefficients_device(d, sp)
            one.append(_native.last_kernel_times(0))
        _native.set_option("stage_times", 0)
        med = {k: sorted(t[k] for t in one)[5] * 1e3 for k in one[0] if k != "h2d_ms"}
        print(f"{w} {opt}={v}: batch {rate(d, sp, ref=ref):6.1f} us/ROI | single-call stages (us) "
              + " ".join(f"{k[:-3]} {t:.1f}" for k, t in med.items()), flush=True)
    _native.set_option(opt, vals[0])
