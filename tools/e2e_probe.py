"""e2e (host batch from pinned memory) ROIs/s vs host options, same process."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import _native  # noqa: E402

K = 40
for w in sys.argv[1:] or ["c2"]:
    rois, _ = bench.load_workload(w)
    m, sp = rois[0]
    h = torch.from_numpy(m).pin_memory().numpy()
    for opts in ({"host_pack": -1}, {"host_pack": 1}, {"host_pack": 0, "host_split": 0},
                 {"host_pack": 0, "host_split": -1}, {"host_crop": 0}):
        for k, v in opts.items():
            _native.set_option(k, v)
        sc.calculate_coefficients_batch([h] * 16, [sp] * 16)
        best = 0.0
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            outs = sc.calculate_coefficients_batch([h] * K, [sp] * K)
            torch.cuda.synchronize()
            best = max(best, K / (time.perf_counter() - t0))
        scan = sorted(o.host_scan_ms for o in outs)[K // 2]
        print(f"{w} {opts}: e2e {best:7.0f} ROIs/s  host {scan:.3f} ms  h2d {outs[-1].h2d_bytes/1e6:.2f} MB",
              flush=True)
        for k in opts:
            _native.set_option(k, {"host_pack": -1, "host_split": -1, "host_crop": 1}[k])
