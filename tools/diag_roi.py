"""Per-stage CUDA-event times (stage_times=2, median of 5 single calls) and the
work counters of one ROI per workload.  usage: diag_roi.py c2 c3 c4 ... [opt=v,...]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import _native  # noqa: E402

opts = {}
ws = []
for a in sys.argv[1:]:
    if "=" in a:
        opts.update({k: int(v) for k, v in (x.split("=") for x in a.split(","))})
    else:
        ws.append(a)
for w in ws or ["c2"]:
    g, sp = bench.workload_params(w)[0]
    d = torch.from_numpy(g()).cuda()
    with _native.thread_options(stage_times=2, **opts):
        sc.calculate_coefficients_device(d, sp)
        kt = {}
        for _ in range(5):
            c = sc.calculate_coefficients_device(d, sp)
            for k, v in _native.last_kernel_times(0).items():
                kt.setdefault(k, []).append(v)
        diag = _native.last_diagnostics(0)
    med = {k: round(statistics.median(v) * 1e3, 1) for k, v in kt.items()}
    print(w, opts or "", "us:", med, flush=True)
    print(w, "diag:", diag, flush=True)
    print(w, "result:", c.to_dict(), flush=True)
