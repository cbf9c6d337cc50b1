"""Generate golden fixtures under tests/golden/ by running the REFERENCE.

The reference (/root/reference/pkg, Python + numba) cannot travel to the GPU
box, so its outputs are frozen here as small committed fixtures:

* golden.json          -- per-case reference records (7 feature keys) plus the
                          exact counts the reference exposes indirectly
                          (triangle_count = mesh.triangles rows, mesh.py:50-52;
                          active cubes restated from _cell_case, mesh.py:103-128)
* masks_small.npz      -- the small masks themselves and their reference vertex
                          sets (xs, ys, zs in the reference's canonical order)
* clouds.npz           -- random coordinate clouds for the diameters() API with
                          the reference's diameters() outputs in golden.json

Large configurations (C1, C2, C5 of SURVEY.md 8) are regenerated on demand by
paper_2510_02894_b200.synth; their mask sha256 is stored so a generator drift
is detected before any comparison.

usage: python tools/make_golden.py [--big]
Needs a writable copy of the reference (numba cache=True); this script makes
one under /tmp/refpkg if it is missing.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import shutil
import sys
import time

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
GOLD = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)

from paper_2510_02894_b200 import synth  # noqa: E402


def ref_module():
    src = "/tmp/refpkg/src"
    if not os.path.isdir(src):
        shutil.copytree("/root/reference/pkg", "/tmp/refpkg")
    sys.path.insert(0, src)
    import shapecore  # noqa: F401

    return shapecore


def active_cubes(arr: np.ndarray) -> int:
    """Count cells with case not in {0, 255} over the padded grid
    (mesh.py:55-65 padding, mesh.py:103-128 case)."""
    p = np.pad((arr != 0).astype(np.uint8), 1)
    s = (p[:-1, :-1, :-1].astype(np.int16) + p[:-1, :-1, 1:] + p[:-1, 1:, :-1] + p[:-1, 1:, 1:]
         + p[1:, :-1, :-1] + p[1:, :-1, 1:] + p[1:, 1:, :-1] + p[1:, 1:, 1:])
    return int(np.count_nonzero((s != 0) & (s != 8)))


def random_mask(rng, max_dim=20, border=True):
    """Same recipe as the reference test helper (pkg/tests/conftest.py:55-76);
    border=False additionally lets occupied voxels touch the grid faces."""
    dims = tuple(int(d) for d in rng.integers(6, max_dim + 1, size=3))
    nx, ny, nz = dims
    arr = np.zeros((nz, ny, nx), dtype=np.uint8)
    lo = 1 if border else 0
    if rng.random() < 0.5:
        sl = (slice(lo, nz - lo), slice(lo, ny - lo), slice(lo, nx - lo))
        shape = tuple(s.stop - s.start for s in sl)
        arr[sl] = (rng.random(shape) < 0.45).astype(np.uint8)
    else:
        zz, yy, xx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        for _ in range(int(rng.integers(1, 4))):
            cx = rng.uniform(2, nx - 3)
            cy = rng.uniform(2, ny - 3)
            cz = rng.uniform(2, nz - 3)
            r = rng.uniform(1.0, min(dims) / 2.0 - 1.5)
            inside = (xx - cx) ** 2 + (yy - cy) ** 2 + (zz - cz) ** 2 <= r * r
            if border:
                arr[1:-1, 1:-1, 1:-1] |= inside[1:-1, 1:-1, 1:-1].astype(np.uint8)
            else:
                arr |= inside.astype(np.uint8)
    if not arr.any():
        arr[nz // 2, ny // 2, nx // 2] = 1
    return arr


def record(sc, arr, spacing, keep_vertices=False):
    nz, ny, nx = arr.shape
    vol = sc.MaskVolume(dims=(nx, ny, nz), spacing=tuple(float(s) for s in spacing),
                        data=np.ascontiguousarray(arr, dtype=np.uint8).reshape(-1))
    feats, _ = sc.extract_features(vol, sc.resolve_backend("parallel"))
    mesh = sc.marching_cubes(vol)
    rec = {
        "spacing": [float(s) for s in spacing],
        "dims": [nx, ny, nz],
        "features": feats.to_dict(),
        "triangle_count": mesh.triangle_count,
        "active_cubes": active_cubes(arr),
        "occupied": int(np.count_nonzero(arr)),
        "sha256": hashlib.sha256(np.ascontiguousarray(arr, dtype=np.uint8).tobytes()).hexdigest(),
    }
    verts = np.column_stack((mesh.xs, mesh.ys, mesh.zs)) if keep_vertices else None
    return rec, verts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also C1/C2/C5 (minutes)")
    args = ap.parse_args()
    sc = ref_module()
    os.makedirs(GOLD, exist_ok=True)
    cases = []
    arrays = {}

    def add(name, arr, spacing, keep_vertices=True):
        rec, verts = record(sc, arr, spacing, keep_vertices)
        rec["name"] = name
        rec["mask_key"] = f"mask_{len(cases)}"
        arrays[rec["mask_key"]] = np.ascontiguousarray(arr, dtype=np.uint8)
        if verts is not None:
            rec["verts_key"] = f"verts_{len(cases)}"
            arrays[rec["verts_key"]] = verts
        cases.append(rec)

    # Known-answer cases from the reference's own tests.
    add("single_voxel", synth.synth_mask("box", (3, 3, 3), lo=(1, 1, 1), hi=(1, 1, 1)), (1, 1, 1))
    add("single_voxel_aniso", synth.synth_mask("box", (3, 3, 3), lo=(1, 1, 1), hi=(1, 1, 1)),
        (0.5, 2.0, 4.0))
    add("block_2x2x2", synth.synth_mask("box", (4, 4, 4), lo=(1, 1, 1), hi=(2, 2, 2)), (1, 1, 1))
    add("readme_sphere_24_r8", synth.synth_mask("sphere", (24, 24, 24), radius=8), (1, 1, 1))
    add("readme_sphere_24_r8_x2", synth.synth_mask("sphere", (24, 24, 24), radius=8), (2, 2, 2))
    add("sphere_40_r15", synth.synth_mask("sphere", (40, 40, 40), radius=15), (1, 1, 1))
    add("ellipsoid_aniso", synth.synth_mask("ellipsoid", (26, 22, 18), semi_axes=(9.0, 7.0, 5.5)),
        (1.0, 0.5, 2.0))
    add("ellipsoid_24_22_20", synth.synth_mask("ellipsoid", (24, 22, 20), semi_axes=(8, 7, 6)),
        (1, 1, 1))
    # Edge cases the boundary must handle.
    add("one_voxel_grid", np.ones((1, 1, 1), np.uint8), (1, 1, 1))
    add("full_block_touching_faces", np.ones((7, 6, 5), np.uint8), (0.7, 1.3, 2.1))
    line = np.zeros((1, 1, 70), np.uint8)
    line[0, 0, 3:61] = 1
    add("line_1x1x70", line, (1, 1, 1))
    add("x_extent_33", np.pad(np.ones((3, 4, 33), np.uint8), ((1, 1), (1, 1), (0, 0))), (1, 1, 1))
    checker = (np.indices((9, 10, 35)).sum(axis=0) % 2).astype(np.uint8)
    add("checkerboard_35", checker, (1, 1, 1))
    # Seeded random masks: the reference recipe plus spacing draws, with and
    # without a clear border, at x extents that are not multiples of 16/32.
    rng = np.random.default_rng(11)
    spacings = [0.5, 0.8, 1.0, 1.25, 3.0, 5.0]
    for i in range(40):
        arr = random_mask(rng, max_dim=20, border=(i % 4 != 3))
        sp = tuple(float(rng.choice(spacings)) for _ in range(3))
        add(f"random_{i}", arr, sp, keep_vertices=(i < 12))
    rng = np.random.default_rng(12)
    for i in range(6):
        arr = random_mask(rng, max_dim=70, border=(i % 2 == 0))
        add(f"random_wide_{i}", arr, (1.0, 1.0, 1.0), keep_vertices=False)

    # Diameters API on raw clouds (pkg/tests/test_acceptance.py:88-99 recipe).
    rng = np.random.default_rng(23)
    clouds = []
    cloud_arrays = {}
    for i in range(100):
        n = int(rng.integers(1, 201))
        if rng.random() < 0.5:
            xs, ys, zs = (rng.integers(0, 16, size=n) * 0.5 for _ in range(3))
        else:
            xs, ys, zs = (np.round(rng.normal(size=n) * 4.0, 2) for _ in range(3))
        cloud_arrays[f"cloud_{i}"] = np.stack([xs, ys, zs]).astype(np.float64)
        clouds.append({"key": f"cloud_{i}", "diameters": list(sc.diameters(xs, ys, zs))})
    for i, n in enumerate((1000, 3000)):
        pts = rng.normal(size=(3, n)) * np.array([[50.0], [30.0], [10.0]])
        pts[2] = np.round(pts[2])  # shared z values -> populated XY planes
        cloud_arrays[f"cloud_big_{i}"] = pts
        clouds.append({"key": f"cloud_big_{i}", "diameters": list(sc.diameters(*pts))})

    big = []
    if args.big:
        specs = [
            ("C1_sphere64_r24", lambda: synth.synth_mask("sphere", (64, 64, 64), radius=24),
             (1.0, 1.0, 1.0)),
            ("C5_thin_slab", lambda: synth.thin_slab(), (0.5, 0.5, 5.0)),
            ("C2_kits_R30", lambda: synth.kits_like(tumor_mm=30.0), (0.8, 0.8, 1.0)),
        ]
        for name, gen, sp in specs:
            t0 = time.time()
            arr = gen()
            rec, _ = record(sc, arr, sp)
            rec["name"] = name
            big.append(rec)
            print(f"{name}: {rec['features']} T={rec['triangle_count']} "
                  f"active={rec['active_cubes']} ({time.time() - t0:.1f}s)", flush=True)
    else:
        old = os.path.join(GOLD, "golden.json")
        if os.path.exists(old):
            big = json.load(open(old)).get("big", [])

    np.savez_compressed(os.path.join(GOLD, "masks_small.npz"), **arrays)
    np.savez_compressed(os.path.join(GOLD, "clouds.npz"), **cloud_arrays)
    with open(os.path.join(GOLD, "golden.json"), "w") as fh:
        json.dump({
            "generator": "tools/make_golden.py (reference shapecore 1.0.0 via numba, "
                         "backend=parallel)",
            "cases": cases, "clouds": clouds, "big": big,
        }, fh, indent=1)
    print(f"{len(cases)} cases, {len(clouds)} clouds, {len(big)} big")


if __name__ == "__main__":
    main()
