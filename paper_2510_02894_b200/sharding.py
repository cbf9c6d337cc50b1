"""Multi-GPU partitioning of the shape-coefficient path.

Two shapes of work shard naturally; nothing else is split:

* ROI batches (C4): independent masks.  `assign_rois` places them on ranks by
  longest-processing-time on an estimated cost; each rank runs its ROIs with
  no data-path collective; the 9-scalar records are gathered once at the end.
* One very large mesh (C3), `slab_sharded_coefficients`: every rank packs the
  mask (global bbox), runs marching cubes over its contiguous share of the cell
  layers only (`sc_shard_mesh`), then the exact integer partials are
  all-reduced (SUM) and the vertex keys all-gathered; every rank evaluates its
  slice of the triangular pair-tile grid and of the planar groups
  (`sc_shard_diameters`), and the four partial squared maxima are combined
  with one all_reduce(MAX) over NCCL / NVLink.  `sharded_coefficients` is the
  one-call form (full marching cubes on every rank, only the pair grid split).

One process per GPU; torch.distributed is plumbing (process group, NCCL
all-reduce), the compute is the C ABI.  The combine logic takes an injectable
`compute` callable so it is tested on CPU with the gloo backend.
"""

from __future__ import annotations

import heapq
import math
from typing import Callable, List, Optional, Sequence, Tuple


# ---- pair-grid ownership (mirrors of the engine's rules) ---------------------
# The shard entry splits the pair grid by the IDENTITY of each unit, not by
# position in a list, so the split is exact whatever order the device's
# atomically compacted work lists come out in.  These restate the rules the
# kernels apply; tests/test_sharding.py runs a CPU shard stub built on them.

CHUNK_3D = 128      # vertices per 3-D chunk (sc_device.cuh kChunk3)
CHUNK_PLANAR = 128  # entries per in-plane chunk (kPlaneChunk)
TILE_PLANAR = 256   # entries per in-plane tile = 2 chunks (planar.cu kPT)


def tile_pair_index(i: int, j: int, n: int) -> int:
    """Row-major index of (i, j), i <= j, in the upper triangle of an n x n
    grid (sc_device.cuh tile_pair is its inverse)."""
    return i * n - i * (i - 1) // 2 + (j - i)


def owner_3d(i: int, j: int, n_chunks: int, nshards: int) -> int:
    """Shard owning 3-D chunk pair (i, j), i <= j: its tile-pair index mod
    nshards (csrc/prune.cu test_chunk_pair, :457)."""
    return tile_pair_index(i, j, n_chunks) % nshards


def owner_planar(p: int, nshards: int) -> int:
    """Shard owning every in-plane chunk pair of plane p (engine plane order:
    XY by z, then XZ by y, then YZ by x): p mod nshards (csrc/planar.cu
    plane_filter).  Whole planes, so no shard depends on the order of a
    plane's entries."""
    return p % nshards


def shard_pairs_3d(n: int, shard: int, nshards: int, chunk: int = CHUNK_3D):
    """Chunk pairs (i, j), i <= j, of n vertices owned by `shard`."""
    C = (n + chunk - 1) // chunk
    for i in range(C):
        for j in range(i, C):
            if owner_3d(i, j, C, nshards) == shard:
                yield i, j


def shard_pairs_planar(plane_sizes: Sequence[int], shard: int, nshards: int,
                       chunk: int = CHUNK_PLANAR, tile: int = TILE_PLANAR):
    """(plane, ci, cj) in-plane chunk pairs, ci <= cj, owned by `shard`.
    Planes in engine order (XY by z, then XZ by y, then YZ by x, ascending);
    a plane with < 2 entries has no tile pairs."""
    u0 = 0
    for p, np_ in enumerate(plane_sizes):
        if np_ < 2:
            continue
        nc = (np_ + chunk - 1) // chunk
        T = (np_ + tile - 1) // tile
        for I in range(T):
            for J in range(I, T):
                u = u0 + tile_pair_index(I, J, T)
                for h in range(2):
                    for b in range(2):
                        i, j = 2 * I + h, 2 * J + b
                        if i < nc and j < nc and j >= i and owner_planar(p, nshards) == shard:
                            yield p, i, j
        u0 += T * (T + 1) // 2


def roi_cost(occupied_voxels: int, voxels: int) -> float:
    """Cost model for LPT: a streaming term for the mask plus the O(V^2)
    diameter term with V ~ surface ~ occupied^(2/3)."""
    v = max(1.0, float(occupied_voxels)) ** (2.0 / 3.0) * 6.0
    return voxels / 6.45e12 * 2 + v * v / 2 / 3e12


def assign_rois(costs: Sequence[float], nranks: int) -> List[List[int]]:
    """Longest-processing-time-first assignment; returns ROI indices per rank
    (each list in ascending index order)."""
    heap = [(0.0, r) for r in range(nranks)]
    heapq.heapify(heap)
    out: List[List[int]] = [[] for _ in range(nranks)]
    for i in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(x) for x in out]


def batch_coefficients(masks: Sequence, spacings: Sequence[Sequence[float]],
                       costs: Optional[Sequence[float]] = None, group=None,
                       compute: Optional[Callable] = None):
    """C4 on the calling rank's GPU: compute the ROIs LPT-assigned to this rank
    and all-gather the records (a list in input order, on every rank)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if costs is None:
        costs = [float(getattr(m, "size", 1)) for m in masks]
    mine = assign_rois(costs, world)[rank]
    if compute is None:
        from .features import calculate_coefficients_batch

        def compute(ms, sps):
            return [c.to_dict() | {"triangle_count": c.triangle_count,
                                   "active_cubes": c.active_cubes}
                    for c in calculate_coefficients_batch(ms, sps)]
    local = compute([masks[i] for i in mine], [spacings[i] for i in mine]) if mine else []
    pairs = list(zip(mine, local))
    if world == 1:
        gathered = [pairs]
    else:
        gathered = [None] * world
        dist.all_gather_object(gathered, pairs, group=group)
    out = [None] * len(masks)
    for part in gathered:
        for i, rec in part:
            out[i] = rec
    return out


def sharded_coefficients(mask, spacing: Sequence[float], group=None,
                         compute: Optional[Callable] = None):
    """One large ROI split across the ranks of `group`: each rank evaluates its
    shard of the pair grid, then one all_reduce(MAX) of the 4 squared maxima.

    compute(shard, nshards, sq4) -> record dict; must write the shard's squared
    maxima into the 4-element float64 tensor sq4 (default: the C ABI)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if compute is None:
        from .features import calculate_coefficients_shard

        def compute(shard, nshards, sq4):
            c = calculate_coefficients_shard(mask, spacing, shard, nshards, sq4)
            return c.to_dict() | {"triangle_count": c.triangle_count,
                                  "active_cubes": c.active_cubes}
        device = mask.device
    else:
        device = torch.device("cpu")
    sq4 = torch.zeros(4, dtype=torch.float64, device=device)
    rec = compute(rank, world, sq4)
    if world > 1:
        dist.all_reduce(sq4, op=dist.ReduceOp.MAX, group=group)
    d = [math.sqrt(v) for v in sq4.cpu().tolist()]
    rec = dict(rec)
    rec.update({"Maximum3DDiameter": d[0], "Maximum2DDiameterXY": d[1],
                "Maximum2DDiameterXZ": d[2], "Maximum2DDiameterYZ": d[3]})
    return rec


# ---- slab split: marching cubes divided too (sc_shard_mesh / _diameters) -----

def exchange_mesh(sums, keys, n_local: int, group=None):
    """The slab split's one data exchange between the two phases: all-reduce
    (SUM) of the int64 partials `sums` in place, and all-gather of every rank's
    first n_local vertex keys (4 int32 each; ragged, padded to the largest
    share).  Returns (gathered keys, their total count)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return keys, n_local
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    cnt = torch.tensor([n_local], dtype=torch.int64, device=sums.device)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    m = max(counts)
    local = keys[: 4 * m] if keys.numel() >= 4 * m else torch.cat(
        [keys, keys.new_zeros(4 * m - keys.numel())])
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local.contiguous(), group=group)
    gathered = torch.cat([p[: 4 * c] for p, c in zip(parts, counts)])
    return gathered, sum(counts)


def slab_sharded_coefficients(mask, spacing: Sequence[float], group=None,
                              mesh: Optional[Callable] = None,
                              diameters: Optional[Callable] = None):
    """One large ROI, marching cubes and pair grid both split across the ranks
    of `group`: phase 1 on this rank's cell layers, one
    exchange (`exchange_mesh`), phase 2 on this rank's pair units, one
    all_reduce(MAX) of the 4 squared maxima.

    mesh(shard, nshards) -> (sums, keys, n_local, bbox) and
    diameters(sums, keys, n_all, bbox, shard, nshards, sq4) -> record dict
    default to the C ABI (device-resident mask); injectable for CPU tests."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if mesh is None:
        from .features import shard_diameters, shard_exchange_sizes, shard_mesh

        shape = tuple(int(d) for d in mask.shape)
        n_sums, key_cap = shard_exchange_sizes(shape)

        def mesh(shard, nshards):
            sums = torch.empty(n_sums, dtype=torch.int64, device=mask.device)
            keys = torch.empty(4 * key_cap, dtype=torch.int32, device=mask.device)
            n, bbox = shard_mesh(mask, spacing, shard, nshards, sums, keys)
            return sums, keys, n, bbox

        def diameters(sums, keys, n_all, bbox, shard, nshards, sq4):
            c = shard_diameters(sums, keys, n_all, shape, bbox, spacing, shard, nshards, sq4)
            return c.to_dict() | {"triangle_count": c.triangle_count,
                                  "active_cubes": c.active_cubes}
        device = mask.device
    else:
        device = torch.device("cpu")
    sums, keys, n_local, bbox = mesh(rank, world)
    keys_all, n_all = exchange_mesh(sums, keys, n_local, group)
    sq4 = torch.zeros(4, dtype=torch.float64, device=device)
    rec = dict(diameters(sums, keys_all, n_all, bbox, rank, world, sq4))
    if world > 1:
        dist.all_reduce(sq4, op=dist.ReduceOp.MAX, group=group)
    d = [math.sqrt(v) for v in sq4.cpu().tolist()]
    rec.update({"Maximum3DDiameter": d[0], "Maximum2DDiameterXY": d[1],
                "Maximum2DDiameterXZ": d[2], "Maximum2DDiameterYZ": d[3]})
    return rec


def simulate_slab_shards(mask, spacing: Sequence[float], nshards: int, timer=None):
    """All `nshards` shards of the slab split run one after another on this
    GPU, the exchange done locally (sum / concatenate): the N-GPU result on 1
    GPU.  timer(phase, shard, fn) may wrap each phase call (bench timing).
    Returns (record, per-shard list of (phase-1 record, phase-2 record))."""
    import torch

    from .features import shard_diameters, shard_exchange_sizes, shard_mesh

    run = timer or (lambda phase, shard, fn: fn())
    shape = tuple(int(d) for d in mask.shape)
    n_sums, key_cap = shard_exchange_sizes(shape)
    tot = torch.zeros(n_sums, dtype=torch.int64, device=mask.device)
    parts, bbox = [], None
    for s in range(nshards):
        sums = torch.empty(n_sums, dtype=torch.int64, device=mask.device)
        keys = torch.empty(4 * key_cap, dtype=torch.int32, device=mask.device)
        n, bb = run(1, s, lambda: shard_mesh(mask, spacing, s, nshards, sums, keys))
        assert bbox is None or bb == bbox
        bbox = bb
        tot += sums
        parts.append(keys[: 4 * n].clone())
    keys_all = torch.cat(parts)
    n_all = keys_all.numel() // 4
    sq = torch.zeros(4, dtype=torch.float64, device=mask.device)
    rec = None
    for s in range(nshards):
        sq4 = torch.zeros(4, dtype=torch.float64, device=mask.device)
        c = run(2, s, lambda: shard_diameters(tot, keys_all, n_all, shape, bbox, spacing, s,
                                              nshards, sq4))
        sq = torch.maximum(sq, sq4)
        rec = c
    d = [math.sqrt(v) for v in sq.cpu().tolist()]
    out = rec.to_dict() | {"triangle_count": rec.triangle_count,
                           "active_cubes": rec.active_cubes}
    out.update({"Maximum3DDiameter": d[0], "Maximum2DDiameterXY": d[1],
                "Maximum2DDiameterXZ": d[2], "Maximum2DDiameterYZ": d[3]})
    return out
