"""Randomized parity stress: N seeded masks of varied shape, size, spacing and
grid alignment through every entry point (host single call, host batch with
crop/split, device batch), compared with the CPU oracle: counts exact,
diameters bit-exact, area/volume within 1e-6 (the north_star bar).

usage: python tools/stress_parity.py [N] [seed0]"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_02894_b200 as sc  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2510_02894_b200 import synth  # noqa: E402

KEYS = ("Maximum3DDiameter", "Maximum2DDiameterXY", "Maximum2DDiameterXZ", "Maximum2DDiameterYZ")


def make(rng):
    kind = rng.integers(0, 5)
    dims = [int(v) for v in rng.integers(2, 120, 3)]
    if rng.random() < 0.3:
        dims[0] = int(rng.choice([32, 64, 96, 128]))  # fast (nx % 32 == 0) pack path
    arr = np.zeros(dims[::-1], dtype=np.uint8)
    if kind == 0:  # random voxels (small grids: every voxel is surface)
        arr = arr[:24, :24, :24].copy()
        arr[rng.random(arr.shape) < rng.uniform(0.001, 0.6)] = 1
    elif kind == 1:  # ellipsoid blobs
        for _ in range(int(rng.integers(1, 9))):
            semi = rng.uniform(0.6, 0.5 * max(dims), 3)
            c = [rng.uniform(-2, dims[a] + 1) for a in range(3)]
            synth.ellipsoid_into(arr, c, semi)
    elif kind == 2:  # thin sheets / lines
        ax = int(rng.integers(0, 3))
        idx = [slice(None)] * 3
        idx[ax] = slice(int(rng.integers(0, arr.shape[ax])), None, int(rng.integers(2, 9)))
        arr[tuple(idx)] = 1
        arr[rng.random(arr.shape) < 0.5] = 0
    elif kind == 3:  # boxes touching the grid faces
        for _ in range(int(rng.integers(1, 4))):
            lo = [int(rng.integers(0, s)) for s in arr.shape]
            hi = [int(rng.integers(l + 1, s + 1)) for l, s in zip(lo, arr.shape)]
            arr[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] = rng.integers(1, 256)
    else:  # single voxels, nonbinary values
        for _ in range(int(rng.integers(1, 5))):
            arr[tuple(int(rng.integers(0, s)) for s in arr.shape)] = rng.integers(1, 256)
    if not arr.any():
        arr[0, 0, 0] = 1
    sp = tuple(float(v) for v in rng.choice([0.3, 0.5, 0.7, 0.8, 1.0, 1.25, 2.0, 3.3, 5.0], 3))
    return arr, sp


def check(got, want, tag):
    rec = got.to_dict()
    assert rec["VertexCount"] == want["VertexCount"], (tag, rec["VertexCount"], want["VertexCount"])
    assert got.triangle_count == want["triangle_count"], tag
    for k in KEYS:
        assert rec[k] == want[k], (tag, k, rec[k], want[k])
    for k in ("MeshVolume", "SurfaceArea"):
        assert abs(rec[k] - want[k]) <= 1e-6 * max(abs(want[k]), 1e-300), (tag, k, rec[k], want[k])


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rng = np.random.default_rng(seed0)
    cases = []
    while len(cases) < n:  # keep the oracle's O(V^2) diameters quick: V <= 40 K
        a, sp = make(rng)
        if oracle.marching_cubes(a, sp).vertex_count <= 40000:
            cases.append((a, sp))
    wants = [oracle.extract_features(a, sp, threads=0) for a, sp in cases]
    for i, ((a, sp), w) in enumerate(zip(cases, wants)):
        check(sc.calculate_coefficients(a, sp), w, ("single", i))
    for i, (o, w) in enumerate(zip(sc.calculate_coefficients_batch([a for a, _ in cases],
                                                                   [sp for _, sp in cases]),
                                   wants)):
        check(o, w, ("host batch", i))
    from paper_2510_02894_b200 import _native
    _native.set_option("host_pack", 1)  # bit volume packed on the host
    _native.set_option("host_split", 0)
    try:
        for i, (o, w) in enumerate(zip(sc.calculate_coefficients_batch(
                [a for a, _ in cases], [sp for _, sp in cases]), wants)):
            check(o, w, ("host-packed batch", i))
    finally:
        _native.set_option("host_pack", -1)
        _native.set_option("host_split", -1)
    ds = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a, _ in cases]
    for i, (o, w) in enumerate(zip(sc.calculate_coefficients_device_batch(
            ds, [sp for _, sp in cases]), wants)):
        check(o, w, ("device batch", i))
    print(f"stress parity ok: {n} masks x 4 entry paths (seed {seed0})")


if __name__ == "__main__":
    main()
