"""Synthetic ROI masks (host, numpy) for tests and benchmarks.

`synth_mask` restates the reference generator (pkg/src/shapecore/volume.py:
220-295): a voxel is occupied iff its integer centre satisfies the analytic
inequality, evaluated in float64.  The large benchmark configurations follow
SURVEY.md Appendix D exactly (C2 `kits_like`, C3 `noisy_ellipsoid`, C5
`thin_slab`, C4 `kits_batch_params`).

All masks are uint8 arrays of shape (nz, ny, nx) -- x fastest, the reference
MaskVolume layout (volume.py:59-66).
"""

from __future__ import annotations

import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .errors import ShapeExceedsBounds


def _check_extent(center, reach, dims) -> None:
    """volume.py:288-295: shapes must keep a 1-voxel background margin."""
    for c, r, n in zip(center, reach, dims):
        if math.ceil(c - r) < 1 or math.floor(c + r) > n - 2:
            raise ShapeExceedsBounds(
                f"extent [{c - r}, {c + r}] breaks the 1-voxel margin in a {n}-voxel axis"
            )


def synth_mask(kind: str, dims: Tuple[int, int, int], *, radius: Optional[float] = None,
               semi_axes: Optional[Sequence[float]] = None,
               center: Optional[Sequence[float]] = None,
               lo: Optional[Sequence[int]] = None,
               hi: Optional[Sequence[int]] = None) -> np.ndarray:
    """Deterministic sphere / ellipsoid / box mask, (nz, ny, nx) uint8."""
    nx, ny, nz = (int(d) for d in dims)
    if min(nx, ny, nz) < 3:
        raise ShapeExceedsBounds(f"dims {dims} leave no room for a 1-voxel margin")
    if center is None:
        center = ((nx - 1) / 2.0, (ny - 1) / 2.0, (nz - 1) / 2.0)
    cx, cy, cz = (float(c) for c in center)
    iz, iy, ix = np.meshgrid(np.arange(nz, dtype=np.float64), np.arange(ny, dtype=np.float64),
                             np.arange(nx, dtype=np.float64), indexing="ij")
    if kind == "sphere":
        if radius is None:
            raise ValueError("sphere needs a radius")
        _check_extent((cx, cy, cz), (radius, radius, radius), (nx, ny, nz))
        occ = (ix - cx) ** 2 + (iy - cy) ** 2 + (iz - cz) ** 2 <= float(radius) ** 2
    elif kind == "ellipsoid":
        if semi_axes is None:
            raise ValueError("ellipsoid needs semi_axes")
        a, b, c = (float(s) for s in semi_axes)
        if min(a, b, c) <= 0:
            raise ValueError(f"semi_axes must be positive, got {semi_axes}")
        _check_extent((cx, cy, cz), (a, b, c), (nx, ny, nz))
        occ = ((ix - cx) / a) ** 2 + ((iy - cy) / b) ** 2 + ((iz - cz) / c) ** 2 <= 1.0
    elif kind == "box":
        if lo is None or hi is None:
            raise ValueError("box needs lo and hi corners")
        lo = tuple(int(v) for v in lo)
        hi = tuple(int(v) for v in hi)
        for axis, (l, h, n) in enumerate(zip(lo, hi, (nx, ny, nz))):
            if l > h:
                raise ValueError(f"box lo {lo} exceeds hi {hi} on axis {axis}")
            if l < 1 or h > n - 2:
                raise ShapeExceedsBounds(f"box [{lo}, {hi}] breaks the 1-voxel margin")
        occ = ((ix >= lo[0]) & (ix <= hi[0]) & (iy >= lo[1]) & (iy <= hi[1])
               & (iz >= lo[2]) & (iz <= hi[2]))
    else:
        raise ValueError(f"unknown shape kind {kind!r}")
    return np.ascontiguousarray(occ, dtype=np.uint8)


def ellipsoid_into(arr: np.ndarray, c, semi) -> None:
    """OR an ellipsoid into arr (nz, ny, nx), restricted to its index box with a
    1-voxel clear border."""
    nz, ny, nx = arr.shape
    lo, hi = [], []
    for ci, si, n in zip(c, semi, (nx, ny, nz)):
        lo.append(max(1, int(math.floor(ci - si))))
        hi.append(min(n - 2, int(math.ceil(ci + si))))
    if any(l > h for l, h in zip(lo, hi)):
        return
    zz, yy, xx = np.ogrid[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1]
    inside = (((xx - c[0]) / semi[0]) ** 2 + ((yy - c[1]) / semi[1]) ** 2
              + ((zz - c[2]) / semi[2]) ** 2 <= 1.0)
    arr[lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1] |= inside.astype(np.uint8)


def kits_like(nx: int = 512, ny: int = 512, nz: int = 600, sp=(0.8, 0.8, 1.0),
              tumor_mm: float = 30.0, kidney_mm=(30.0, 25.0, 55.0)) -> np.ndarray:
    """C2: two kidney ellipsoids plus a tumour sphere."""
    arr = np.zeros((nz, ny, nx), dtype=np.uint8)
    semi = (kidney_mm[0] / sp[0], kidney_mm[1] / sp[1], kidney_mm[2] / sp[2])
    ellipsoid_into(arr, (0.30 * nx, 0.55 * ny, 0.50 * nz), semi)
    ellipsoid_into(arr, (0.70 * nx, 0.55 * ny, 0.47 * nz), semi)
    t = (0.70 * nx + 25.0 / sp[0], 0.55 * ny, 0.47 * nz + 30.0 / sp[2])
    ellipsoid_into(arr, t, (tumor_mm / sp[0], tumor_mm / sp[1], tumor_mm / sp[2]))
    return arr


def noisy_ellipsoid(n: int = 512, sigma: float = 0.02, seed: int = 1234) -> np.ndarray:
    """C3: ellipsoid with a noisy boundary, r^2 <= 1 + sigma*u (Appendix D)."""
    rng = np.random.default_rng(seed)
    c = (n - 1) / 2.0
    a, b, cc = 0.45 * n, 0.38 * n, 0.32 * n
    u = rng.uniform(-1.0, 1.0, size=(n, n, n))
    arr = np.empty((n, n, n), dtype=np.uint8)
    x = (np.arange(n, dtype=np.float64) - c) / a
    y = (np.arange(n, dtype=np.float64) - c) / b
    for iz in range(n):  # slice-wise to bound memory; same arithmetic
        z = (iz - c) / cc
        r2 = x[None, :] ** 2 + y[:, None] ** 2 + z ** 2
        arr[iz] = r2 <= 1.0 + sigma * u[iz]
    arr[0] = arr[-1] = 0
    arr[:, 0] = arr[:, -1] = 0
    arr[:, :, 0] = arr[:, :, -1] = 0
    return arr


def thin_slab(nx: int = 512, ny: int = 512, nz: int = 24, blobs: int = 400,
              seed: int = 7) -> np.ndarray:
    """C5: many small anisotropic blobs in a thin slab (Appendix D); use with
    spacing (0.5, 0.5, 5.0)."""
    rng = np.random.default_rng(seed)
    arr = np.zeros((nz, ny, nx), dtype=np.uint8)
    for _ in range(blobs):
        a, b = rng.uniform(2, 10, 2)
        c = rng.uniform(0.6, 2.5)
        cx = rng.uniform(12, nx - 13)
        cy = rng.uniform(12, ny - 13)
        cz = rng.uniform(3, nz - 4)
        ellipsoid_into(arr, (cx, cy, cz), (a, b, c))
    return arr


def kits_batch_params(count: int = 300, seed: int = 2025) -> List[dict]:
    """C4: seeded draw of varied KiTS-like masks."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        nz = int(rng.integers(200, 701))
        inplane = float(rng.uniform(0.6, 0.9))
        jitter = rng.uniform(0.8, 1.2, size=3)
        tumor = float(rng.uniform(10.0, 75.0))
        out.append({
            "nx": 512, "ny": 512, "nz": nz,
            "sp": (inplane, inplane, 1.0),
            "kidney_mm": tuple(float(v) for v in np.array([30.0, 25.0, 55.0]) * jitter),
            "tumor_mm": tumor,
        })
    return out


def kits_from_params(p: dict) -> np.ndarray:
    return kits_like(p["nx"], p["ny"], p["nz"], p["sp"], p["tumor_mm"], p["kidney_mm"])
