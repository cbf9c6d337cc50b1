"""Device-batch throughput (us per ROI, CUDA events) of one workload under
several option sets.  usage: batch_probe.py <workload> <B> "opt=v,opt=v" ...
('-' = defaults).  Masks cycle through the workload's ROIs (all in HBM)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import _native  # noqa: E402

w, B = sys.argv[1], int(sys.argv[2])
gens = bench.workload_params(w)
dm = [torch.from_numpy(g()).cuda() for g, _ in gens]
sps = [sp for _, sp in gens]
ms = [dm[i % len(dm)] for i in range(B)]
ss = [sps[i % len(sps)] for i in range(B)]
s = torch.cuda.Stream()
ref = [c.to_dict() for c in sc.calculate_coefficients_device_batch(ms, ss, stream=s)]
for spec in sys.argv[3:] or ["-"]:
    opts = {} if spec == "-" else {k: int(v) for k, v in (x.split("=") for x in spec.split(","))}
    with _native.thread_options(**opts):
        best = []
        for r in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            try:
                out = sc.calculate_coefficients_device_batch(ms, ss, stream=s)
            except Exception:  # timing-only option sets (debug cuts) may not produce records
                out = []
            e1.record(s)
            torch.cuda.synchronize()
            if r:
                best.append(e0.elapsed_time(e1) * 1e3 / B)
        ok = [c.to_dict() for c in out] == ref
    print(f"{w} B={B} {spec:40s} {min(best):7.2f} us/ROI (runs {', '.join(f'{x:.2f}' for x in best)})"
          f"{'' if ok else '  RESULTS DIFFER'}", flush=True)
