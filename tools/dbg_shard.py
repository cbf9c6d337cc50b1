"""Shard entry vs full call on one workload: per-shard squared maxima and
work counters, pruned and unpruned.  usage: dbg_shard.py [workload] [N ...]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import _native  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c3"
ns = [int(v) for v in sys.argv[2:]] or [2]
rois, _ = bench.load_workload(w)
m, sp = rois[0]
d = torch.from_numpy(m).cuda()
for prune in (1, 0):
    with _native.thread_options(prune=prune):
        full = sc.calculate_coefficients_device(d, sp)
        print(f"prune={prune} full d3={full.max_3d_diameter!r} sq={full.max_3d_diameter ** 2!r}",
              _native.last_diagnostics(0), flush=True)
        sq = torch.zeros(4, dtype=torch.float64, device="cuda")
        for n in ns:
            for s in range(n):
                part = sc.calculate_coefficients_shard(d, sp, s, n, sq)
                v = sq.cpu().tolist()
                print(f"  N={n} shard {s}: sq3={v[0]!r} d3={math.sqrt(v[0])!r} part={part.max_3d_diameter!r}",
                      _native.last_diagnostics(0), flush=True)
