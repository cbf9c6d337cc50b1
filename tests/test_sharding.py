"""Multi-rank host logic on CPU (gloo, world_size 2): ROI-batch assignment and
the pair-grid shard + all_reduce(MAX) combine.  The per-shard compute is a CPU
stub that follows the engine's partition exactly -- ownership by unit identity
(sharding.owner_3d = prune.cu test_chunk_pair, sharding.owner_planar = planar.cu plane_filter) --
with the reference's pair arithmetic (features.py:140-148)."""

import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2510_02894_b200.sharding import (assign_rois, owner_3d, shard_pairs_3d,
                                            shard_pairs_planar, tile_pair_index)


def test_identity_ownership_partitions_every_pair_once():
    for n in (1, 2, 127, 128, 129, 1000, 5000):
        C = (n + 127) // 128
        all_pairs = [(i, j) for i in range(C) for j in range(i, C)]
        for g in (1, 2, 3, 4, 8):
            got = sorted(p for s in range(g) for p in shard_pairs_3d(n, s, g))
            assert got == all_pairs
            assert [tile_pair_index(i, j, C) for i, j in all_pairs] == list(range(len(all_pairs)))
            if len(all_pairs) >= g:  # balanced: shard sizes differ by <= 1
                sizes = [sum(1 for _ in shard_pairs_3d(n, s, g)) for s in range(g)]
                assert max(sizes) - min(sizes) <= 1
    sizes = [0, 1, 2, 127, 128, 129, 255, 256, 257, 600, 1]
    want = []
    for p, m in enumerate(sizes):
        nc = (m + 127) // 128 if m >= 2 else 0
        want += [(p, i, j) for i in range(nc) for j in range(i, nc)]
    for g in (1, 2, 3, 4, 8):
        got = sorted(t for s in range(g) for t in shard_pairs_planar(sizes, s, g))
        assert got == sorted(want), g
    assert owner_3d(0, 0, 5, 4) == 0 and owner_3d(1, 1, 5, 4) == 5 % 4


def test_lpt_assignment_balanced_and_complete():
    rng = np.random.default_rng(2025)
    costs = list(rng.uniform(1, 100, size=300))
    for g in (1, 2, 4, 8):
        parts = assign_rois(costs, g)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(300))
        loads = [sum(costs[i] for i in p) for p in parts]
        assert max(loads) <= sum(costs) / g + max(costs)  # LPT bound


def _planes(key):
    """Engine plane order within one family: ascending key."""
    return sorted(set(key.tolist()))


def _shard_stub(pts, chunk=8):
    """CPU stand-in for sc_calculate_coefficients_shard on a point set: squared
    maxima over this shard's 3-D chunk pairs and planar chunk pairs, owned by
    identity as on the device (small chunks so the grid has many units)."""
    xs, ys, zs = pts
    n = len(xs)

    def sq_max(ii, jj, cols):
        d = 0.0
        for c in cols:
            diff = c[jj][None, :] - c[ii][:, None]
            d = d + diff * diff
        return float(np.max(d)) if np.size(d) else 0.0

    def compute(shard, nshards, sq4):
        m3 = 0.0
        for i, j in shard_pairs_3d(n, shard, nshards, chunk=chunk):
            ii = np.arange(i * chunk, min(n, (i + 1) * chunk))
            jj = np.arange(j * chunk, min(n, (j + 1) * chunk))
            m3 = max(m3, sq_max(ii, jj, (xs, ys, zs)))
        # planes: XY (same z), XZ (same y), YZ (same x), each family in key order
        fams = ((zs, (xs, ys)), (ys, (xs, zs)), (xs, (ys, zs)))
        members, sizes, fam_of = [], [], []
        for f, (key, _) in enumerate(fams):
            for k in _planes(key):
                idx = np.flatnonzero(key == k)
                members.append(idx)
                sizes.append(len(idx))
                fam_of.append(f)
        planar = [0.0, 0.0, 0.0]
        for p, i, j in shard_pairs_planar(sizes, shard, nshards, chunk=chunk, tile=2 * chunk):
            idx = members[p]
            ii, jj = idx[i * chunk:(i + 1) * chunk], idx[j * chunk:(j + 1) * chunk]
            f = fam_of[p]
            planar[f] = max(planar[f], sq_max(ii, jj, fams[f][1]))
        sq4[0], sq4[1], sq4[2], sq4[3] = m3, planar[0], planar[1], planar[2]
        return {"VertexCount": n}

    return compute


def test_identity_shards_combine_to_the_full_maxima(oracle_mod):
    """Sequential shards + MAX == the reference's diameters, for N = 1..8."""
    import torch

    rng = np.random.default_rng(11)
    n = 300
    pts = tuple((rng.integers(0, 12, size=n) * 0.5).astype(np.float64) for _ in range(3))
    want = oracle_mod.diameters(*pts)
    for g in (1, 2, 3, 4, 8):
        acc = np.zeros(4)
        for s in range(g):
            sq4 = torch.zeros(4, dtype=torch.float64)
            _shard_stub(pts)(s, g, sq4)
            acc = np.maximum(acc, sq4.numpy())
        assert tuple(math.sqrt(v) for v in acc) == tuple(want), g


def _worker(rank, world, port, pts, want, q):
    import torch.distributed as dist

    from paper_2510_02894_b200 import sharding

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rec = sharding.sharded_coefficients(None, (1, 1, 1), compute=_shard_stub(pts))
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


# ---- slab split: the exchange between the two phases (gloo, world 3) ---------

def _slab_parts(shard):
    """Shard-local phase-1 output of the CPU stub: int64 partials and a ragged
    key share (shard 1 has none)."""
    import torch

    g = torch.Generator().manual_seed(100 + shard)
    sums = torch.randint(0, 1 << 40, (37,), generator=g, dtype=torch.int64)
    n = (0, 5, 3)[shard]
    keys = torch.arange(4 * n, dtype=torch.int32) + 1000 * shard
    pad = torch.full((4 * 7,), -1, dtype=torch.int32)  # a key buffer larger than the share
    pad[: 4 * n] = keys
    return sums, pad, n


def _slab_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2510_02894_b200 import sharding

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        want_sums = sum(_slab_parts(s)[0] for s in range(world))
        want_keys = torch.cat([_slab_parts(s)[1][: 4 * _slab_parts(s)[2]] for s in range(world)])
        seen = {}

        def mesh(shard, nshards):
            assert (shard, nshards) == (rank, world)
            sums, keys, n = _slab_parts(shard)
            return sums.clone(), keys, n, (1, 2, 3, 4, 5, 6)

        def diameters(sums, keys, n_all, bbox, shard, nshards, sq4):
            seen["ok"] = (torch.equal(sums, want_sums) and n_all == want_keys.numel() // 4
                          and torch.equal(keys[: 4 * n_all], want_keys)
                          and bbox == (1, 2, 3, 4, 5, 6))
            sq4.copy_(torch.tensor([1.0 + shard, 4.0 - shard, 9.0, 16.0 * (shard == 1)],
                                   dtype=torch.float64))
            return {"VertexCount": n_all}

        rec = sharding.slab_sharded_coefficients(None, (1, 1, 1), mesh=mesh, diameters=diameters)
        got = [rec[k] for k in ("Maximum3DDiameter", "Maximum2DDiameterXY",
                                "Maximum2DDiameterXZ", "Maximum2DDiameterYZ")]
        q.put((rank, seen.get("ok", False), got, rec["VertexCount"]))
    finally:
        dist.destroy_process_group()


def test_gloo_world3_slab_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, got, nv in res:
        assert ok, f"rank {rank}: summed partials / gathered keys differ"
        assert got == [math.sqrt(3.0), 2.0, 3.0, 4.0]
        assert nv == 8
