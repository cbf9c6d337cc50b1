"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
C1 and C5 plus a small KiTS-like mask through every entry -- single host call,
device call, host batch (crop / split / host pack), device batch (32 slots,
pack chain, TMA pack), shard entry, two-phase slab split, raw typed payloads (C and Fortran), mesh
export, diameters -- and checks the results agree.  Small sizes: the tools
slow kernels down by 10-100x.  usage: sanitize_run.py [quick]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import _native, sharding, synth  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
cases = [(synth.synth_mask("sphere", (64, 64, 64), radius=24), (1.0, 1.0, 1.0)),
         (synth.kits_like(128, 128, 96, (0.8, 0.8, 1.0), 20.0), (0.8, 0.8, 1.0))]
if not quick:
    cases.append((synth.thin_slab(), (0.5, 0.5, 5.0)))
want = [sc.calculate_coefficients(a, sp).to_dict() for a, sp in cases]
ds = [torch.from_numpy(a).cuda() for a, _ in cases]
for (a, sp), d, w in zip(cases, ds, want):
    assert sc.calculate_coefficients_device(d, sp).to_dict() == w
    sq = torch.zeros(4, dtype=torch.float64, device="cuda")
    best = torch.zeros(4, dtype=torch.float64, device="cuda")
    for s in range(2):
        sc.calculate_coefficients_shard(d, sp, s, 2, sq)
        torch.maximum(best, sq, out=best)
    assert abs(best[0].item() ** 0.5 - w["Maximum3DDiameter"]) == 0.0
    # two-phase slab split (sc_shard_mesh / sc_shard_diameters), 3 shards
    rec = sharding.simulate_slab_shards(d, sp, 3)
    assert all(rec[k] == w[k] for k in w), (rec, w)
got = sc.calculate_coefficients_device_batch(ds * 3, [sp for _, sp in cases] * 3)
assert [g.to_dict() for g in got] == want * 3
for opts in ({}, {"host_pack": 1}, {"host_split": 30}, {"host_crop": 0}):
    with _native.thread_options(**opts):
        got = sc.calculate_coefficients_batch([a for a, _ in cases], [sp for _, sp in cases])
        assert [g.to_dict() for g in got] == want, opts
pays = [(a.astype(np.int16) * 2, None) for a, _ in cases] + \
       [(np.asfortranarray(a.astype(np.float32)), 1.0) for a, _ in cases]
got = sc.coefficients_from_payloads(pays, [sp for _, sp in cases] * 2)
assert [g.to_dict() for g in got] == want * 2
with _native.thread_options(pack_tma=0, pack_chain=0, fused_bbox=0, slots=4):
    got = sc.calculate_coefficients_device_batch(ds, [sp for _, sp in cases])
    assert [g.to_dict() for g in got] == want
m = sc.marching_cubes(sc.MaskVolume.from_array(cases[0][0], cases[0][1]))
assert m.vertex_count == want[0]["VertexCount"]
sc.diameters(m.xs, m.ys, m.zs)
torch.cuda.synchronize()
print("sanitize workload ok:", _native.load().sc_launch_count(), "library kernel launches", flush=True)
