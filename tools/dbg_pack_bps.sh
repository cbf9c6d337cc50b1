#!/bin/bash
# Batch throughput vs pack blocks/SM (SC_PACK_BPS) on C2/C5.
for b in 8 6 4 2; do
  SC_PACK_BPS=$b python - <<'PY'
import os, sys, time
sys.path.insert(0, '.')
import torch, bench
import paper_2510_02894_b200 as sc
from paper_2510_02894_b200 import _native
for w in ("c2", "c5"):
    rois, _ = bench.load_workload(w)
    m, sp = rois[0]
    d = torch.from_numpy(m).cuda()
    ts = []
    for _ in range(10):
        sc.calculate_coefficients_device(d, sp)
        ts.append(_native.last_kernel_times(0))
    pk = sorted(t["pack_ms"] for t in ts)[5] * 1e3
    sc.calculate_coefficients_device_batch([d] * 16, [sp] * 16)
    best = 0
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        sc.calculate_coefficients_device_batch([d] * 100, [sp] * 100)
        torch.cuda.synchronize(); best = max(best, 100 / (time.perf_counter() - t0))
    print("bps", os.environ["SC_PACK_BPS"], w, f"pack {pk:.1f} us batch {best:.0f} ROIs/s", flush=True)
PY
done
