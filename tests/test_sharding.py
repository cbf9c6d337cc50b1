"""Multi-rank host logic on CPU (gloo, world_size 2): ROI-batch assignment and
the pair-grid shard + all_reduce(MAX) combine.  The per-shard compute is a CPU
stub that follows the C engine's partition exactly (shard_range over the
triangular tile grid), with the oracle's reference-arithmetic pair loop."""

import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2510_02894_b200.sharding import assign_rois, shard_range


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 5, 17, 1000, 123457):
        for g in (1, 2, 3, 4, 8):
            spans = [shard_range(n, s, g) for s in range(g)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_lpt_assignment_balanced_and_complete():
    rng = np.random.default_rng(2025)
    costs = list(rng.uniform(1, 100, size=300))
    for g in (1, 2, 4, 8):
        parts = assign_rois(costs, g)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(300))
        loads = [sum(costs[i] for i in p) for p in parts]
        assert max(loads) <= sum(costs) / g + max(costs)  # LPT bound


def _tile_pairs(T):
    return [(i, j) for i in range(T) for j in range(i, T)]


def _shard_stub(pts, tile):
    """CPU stand-in for sc_calculate_coefficients_shard: squared maxima over
    this shard's tile pairs (3-D) and planes (planar), reference arithmetic."""
    from oracle import oracle

    xs, ys, zs = pts

    def compute(shard, nshards, sq4):
        n = len(xs)
        T = (n + tile - 1) // tile
        items = _tile_pairs(T)
        a, b = shard_range(len(items), shard, nshards)
        m3 = 0.0
        for (I, J) in items[a:b]:
            ii = np.arange(I * tile, min(n, (I + 1) * tile))
            jj = np.arange(J * tile, min(n, (J + 1) * tile))
            dx = xs[jj][None, :] - xs[ii][:, None]
            dy = ys[jj][None, :] - ys[ii][:, None]
            dz = zs[jj][None, :] - zs[ii][:, None]
            m3 = max(m3, float((dx * dx + dy * dy + dz * dz).max()))
        planar = []
        for key, (u, v) in ((zs, (xs, ys)), (ys, (xs, zs)), (xs, (ys, zs))):
            planes = sorted(set(key.tolist()))
            pa, pb = shard_range(len(planes), shard, nshards)
            best = 0.0
            for p in planes[pa:pb]:
                sel = key == p
                if sel.sum() >= 2:
                    best = max(best, oracle.diameters(u[sel], v[sel], np.zeros(sel.sum()))[0] ** 2)
            planar.append(best)
        sq4[0], sq4[1], sq4[2], sq4[3] = m3, planar[0], planar[1], planar[2]
        return {"VertexCount": n}

    return compute


def _worker(rank, world, port, pts, want, q):
    import torch.distributed as dist

    from paper_2510_02894_b200 import sharding

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rec = sharding.sharded_coefficients(None, (1, 1, 1), compute=_shard_stub(pts, tile=16))
        got = [rec[k] for k in ("Maximum3DDiameter", "Maximum2DDiameterXY",
                                "Maximum2DDiameterXZ", "Maximum2DDiameterYZ")]
        costs = [float(c) for c in range(1, 11)]
        masks = list(range(10))
        out = sharding.batch_coefficients(masks, [(1, 1, 1)] * 10, costs=costs,
                                          compute=lambda ms, sps: [{"id": m, "rank": rank}
                                                                   for m in ms])
        q.put((rank, got == list(want), [o["id"] for o in out], sorted({o["rank"] for o in out})))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_gloo_world2_sharded_max_and_batch(oracle_mod):
    rng = np.random.default_rng(9)
    n = 150
    pts = tuple((rng.integers(0, 24, size=n) * 0.5).astype(np.float64) for _ in range(3))
    want = oracle_mod.diameters(*pts)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, pts, want, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, ids, ranks in res:
        assert ok, "sharded max != full max"
        assert ids == list(range(10))
        assert ranks == [0, 1]  # both ranks did work
