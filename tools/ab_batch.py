"""A/B of one option on the pipelined device batch (bench `value` path).

usage: ab_batch.py OPTION v1,v2,.. [workloads...] [--k K]
Per workload the masks are staged in HBM once; for each option value the same
K-ROI batch (cycling the workload's distinct masks) runs 3 times, best us/ROI
is printed, and every value's results must equal the first value's.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import _native  # noqa: E402

args = sys.argv[1:]
K = 200
if "--k" in args:
    i = args.index("--k")
    K = int(args[i + 1])
    del args[i:i + 2]
opt, vals = args[0], [int(v) for v in args[1].split(",")]
for kv in filter(None, os.environ.get("SC_OPTS", "").split(",")):
    k, v = kv.split("=")
    _native.set_option(k, int(v))
for w in args[2:] or ["c2", "c4"]:
    rois, _ = bench.load_workload(w)
    dm = [torch.from_numpy(m).cuda() for m, _ in rois]
    sps = [sp for _, sp in rois]
    ms = [dm[i % len(dm)] for i in range(K)]
    ss = [sps[i % len(sps)] for i in range(K)]
    ref = None
    for v in vals:
        _native.set_option(opt, v)
        try:
            outs = sc.calculate_coefficients_device_batch(ms, ss)
        except Exception as exc:  # debug options (AB_NOCHECK) may leave ROIs "empty"
            if not os.environ.get("AB_NOCHECK"):
                raise
            outs = []
        got = [o.to_dict() for o in outs]
        if ref is None:
            ref = got
        if not os.environ.get("AB_NOCHECK"):  # debug options give invalid results
            assert got == ref, (w, opt, v, "results differ")
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            try:
                sc.calculate_coefficients_device_batch(ms, ss)
            except Exception:
                if not os.environ.get("AB_NOCHECK"):
                    raise
            torch.cuda.synchronize()
            best = min(best, (time.perf_counter() - t0) / K * 1e6)
        print(f"{w} {opt}={v}: {best:7.2f} us/ROI  {1e6 / best:9.0f} ROIs/s (K={K})", flush=True)
    _native.set_option(opt, vals[0])
    del dm, ms
    torch.cuda.empty_cache()
