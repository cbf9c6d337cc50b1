"""Shape features on the B200: the reference API over the C ABI.

Mirrors reference pkg/src/shapecore/features.py: `FEATURE_KEYS` (:27-35),
`ShapeFeatures` (:38-60), `extract_features` (:224-265), `diameters` /
`diameters_parallel` (:205-221).  `calculate_coefficients(mask, spacing)` is
the north_star entry (PyRadiomics cShape.calculate_coefficients); it returns
the same 7-key record plus the exact triangle and active-cube counts.

Every call goes to libshapecore_b200.so (hand-written sm_100a kernels).  There
is one implementation: no backend dispatch and no CPU fallback.  `selection`
arguments are accepted for signature compatibility with the reference and
are otherwise ignored.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple, Union

import numpy as np

from . import _native
from .errors import NoVertices
from .timing import StageTimings, now_ms
from .volume import MaskVolume, _check_spacing

FEATURE_KEYS = (
    "MeshVolume",
    "SurfaceArea",
    "Maximum3DDiameter",
    "Maximum2DDiameterXY",
    "Maximum2DDiameterXZ",
    "Maximum2DDiameterYZ",
    "VertexCount",
)


@dataclass(frozen=True)
class ShapeFeatures:
    """The five shape scalars plus the vertex count (features.py:38-60)."""

    mesh_volume: float
    surface_area: float
    max_3d_diameter: float
    max_2d_diameter_xy: float
    max_2d_diameter_xz: float
    max_2d_diameter_yz: float
    vertex_count: int

    def to_dict(self) -> Dict[str, Union[float, int]]:
        return {
            "MeshVolume": self.mesh_volume,
            "SurfaceArea": self.surface_area,
            "Maximum3DDiameter": self.max_3d_diameter,
            "Maximum2DDiameterXY": self.max_2d_diameter_xy,
            "Maximum2DDiameterXZ": self.max_2d_diameter_xz,
            "Maximum2DDiameterYZ": self.max_2d_diameter_yz,
            "VertexCount": self.vertex_count,
        }


@dataclass(frozen=True)
class Coefficients(ShapeFeatures):
    """ShapeFeatures plus the exact counts and stage times of the B200 run."""

    triangle_count: int = 0
    active_cubes: int = 0
    h2d_ms: float = 0.0
    mesh_ms: float = 0.0
    diameters_ms: float = 0.0
    total_ms: float = 0.0
    h2d_bytes: int = 0  # host entries: bytes of the occupied slab copied H2D
    host_scan_ms: float = 0.0  # host scan that found the slab


# Coefficients field <- sc_coeffs field (same names; ctypes already returns
# Python int / float for c_int64 / c_double).
_STRUCT_FIELDS = tuple(name for name, _ in _native.ScCoeffs._fields_)


def _check_spacings(spacings, n: int) -> np.ndarray:
    """Vectorised volume.py:94-101 check of n spacings -> flat float64 (3n)."""
    try:
        sp = np.asarray(spacings, dtype=np.float64)
    except (TypeError, ValueError):
        sp = None
    if sp is None or sp.shape != (n, 3) or not (np.isfinite(sp).all() and (sp > 0).all()):
        for s in spacings:  # the scalar check raises the reference's error
            _check_spacing(s)
        if len(spacings) != n:
            raise ValueError(f"{len(spacings)} spacings for {n} masks")
    return np.ascontiguousarray(sp, dtype=np.float64).reshape(-1)


_STRUCT_DTYPE = np.dtype([(name, "<i8" if t is ctypes.c_int64 else "<f8")
                          for name, t in _native.ScCoeffs._fields_])
assert _STRUCT_DTYPE.itemsize == ctypes.sizeof(_native.ScCoeffs)


def _record(values) -> Coefficients:
    # Batches convert hundreds of records inside timed regions: fill the frozen
    # dataclass's __dict__ directly (what its generated __init__ does, minus
    # one object.__setattr__ call per field).
    rec = object.__new__(Coefficients)
    rec.__dict__.update(zip(_STRUCT_FIELDS, values))
    return rec


def _from_struct(c: _native.ScCoeffs) -> Coefficients:
    return _record(getattr(c, k) for k in _STRUCT_FIELDS)


def _from_structs(outs) -> List[Coefficients]:
    """An sc_coeffs array -> records (one numpy pass over the C array)."""
    return [_record(row) for row in np.frombuffer(outs, dtype=_STRUCT_DTYPE).tolist()]


def _as_mask(mask) -> Tuple[np.ndarray, Tuple[int, int, int]]:
    """(nz, ny, nx) array or MaskVolume -> contiguous uint8 host buffer + dims."""
    if isinstance(mask, MaskVolume):
        return np.ascontiguousarray(mask.data, dtype=np.uint8), tuple(mask.dims)
    arr = np.asarray(mask)
    if arr.ndim != 3:
        raise ValueError(f"mask array must be 3-D (nz, ny, nx), got {arr.ndim}-D")
    if arr.dtype == np.bool_:
        arr = arr.view(np.uint8)
    elif arr.dtype != np.uint8:
        arr = (arr != 0).astype(np.uint8)
    arr = np.ascontiguousarray(arr)
    nz, ny, nx = arr.shape
    return arr.reshape(-1), (nx, ny, nz)


def calculate_coefficients(mask, spacing: Optional[Sequence[float]] = None,
                           device: int = 0) -> Coefficients:
    """Full shape coefficients of a host mask ((nz, ny, nx) array or MaskVolume).

    `spacing` defaults to the MaskVolume's own spacing, else (1, 1, 1) mm.
    Raises EmptyRoi for an all-background mask and NonPositiveSpacing for a
    bad spacing, as the reference does (mesh.py:78-79, volume.py:94-101).
    """
    if spacing is None:
        spacing = mask.spacing if isinstance(mask, MaskVolume) else (1.0, 1.0, 1.0)
    sp = np.asarray(_check_spacing(spacing), dtype=np.float64)
    data, (nx, ny, nz) = _as_mask(mask)
    lib = _native.load()
    out = _native.ScCoeffs()
    rc = lib.sc_calculate_coefficients(
        data.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), nx, ny, nz,
        sp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(device), ctypes.byref(out))
    _native.raise_for(rc, "sc_calculate_coefficients")
    return _from_struct(out)


def _stream_handle(tensor, stream) -> int:
    """cudaStream_t of `stream`, default torch's current stream on the tensor's
    device (0 = the legacy default stream, which the library orders against)."""
    if stream is None:
        import torch

        stream = torch.cuda.current_stream(tensor.device)
    return int(stream.cuda_stream)


def calculate_coefficients_device(mask, spacing: Sequence[float], stream=None) -> Coefficients:
    """Coefficients of a device-resident mask: a CUDA uint8 tensor (nz, ny, nx)
    on the current device (torch is plumbing only: pointer + stream), ordered
    after prior work on `stream` (default: torch's current stream)."""
    sp = np.asarray(_check_spacing(spacing), dtype=np.float64)
    nz, ny, nx = (int(d) for d in mask.shape)
    if not mask.is_contiguous():
        raise ValueError("device mask must be contiguous")
    handle = _stream_handle(mask, stream)
    out = _native.ScCoeffs()
    rc = _native.load().sc_calculate_coefficients_device(
        ctypes.c_void_p(mask.data_ptr()), nx, ny, nz,
        sp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.c_void_p(handle),
        ctypes.byref(out))
    _native.raise_for(rc, "sc_calculate_coefficients_device")
    return _from_struct(out)


def calculate_coefficients_shard(mask, spacing: Sequence[float], shard: int, nshards: int,
                                 sq4, stream=None) -> Coefficients:
    """One shard of the pair grid of a device-resident mask.

    `sq4` is a CUDA float64 tensor of 4 elements that receives this shard's
    squared maxima (3d, xy, xz, yz) for an all_reduce(MAX) across ranks."""
    sp = np.asarray(_check_spacing(spacing), dtype=np.float64)
    nz, ny, nx = (int(d) for d in mask.shape)
    handle = _stream_handle(mask, stream)
    out = _native.ScCoeffs()
    rc = _native.load().sc_calculate_coefficients_shard(
        ctypes.c_void_p(mask.data_ptr()), nx, ny, nz,
        sp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.c_void_p(handle),
        int(shard), int(nshards), ctypes.c_void_p(sq4.data_ptr()), ctypes.byref(out))
    _native.raise_for(rc, "sc_calculate_coefficients_shard")
    return _from_struct(out)


def shard_exchange_sizes(shape) -> Tuple[int, int]:
    """(n_sums, key_cap) of the two-phase shard entry for a (nz, ny, nx) grid:
    int64 elements of the partial-sums vector and vertex capacity of a key
    buffer (4 int32 per vertex)."""
    nz, ny, nx = (int(d) for d in shape)
    n_sums, key_cap = ctypes.c_int64(), ctypes.c_int64()
    rc = _native.load().sc_shard_exchange_sizes(nx, ny, nz, ctypes.byref(n_sums),
                                                 ctypes.byref(key_cap))
    _native.raise_for(rc, "sc_shard_exchange_sizes")
    return int(n_sums.value), int(key_cap.value)


def shard_mesh(mask, spacing: Sequence[float], shard: int, nshards: int, sums, keys,
               stream=None) -> Tuple[int, Tuple[int, ...]]:
    """Phase 1 of the slab-split shard (sc_shard_mesh): marching cubes over the
    shard's share of the cell layers of a device-resident mask.  `sums` (CUDA
    int64, n_sums) receives the exact integer partials to all-reduce(SUM);
    `keys` (CUDA int32, 4 x key_cap) the shard's vertex keys to all-gather.
    Returns (vertex count of the shard, global bbox)."""
    sp = np.asarray(_check_spacing(spacing), dtype=np.float64)
    nz, ny, nx = (int(d) for d in mask.shape)
    if not mask.is_contiguous():
        raise ValueError("device mask must be contiguous")
    handle = _stream_handle(mask, stream)
    n = ctypes.c_int64()
    bbox = (ctypes.c_int32 * 6)()
    rc = _native.load().sc_shard_mesh(
        ctypes.c_void_p(mask.data_ptr()), nx, ny, nz,
        sp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.c_void_p(handle),
        int(shard), int(nshards), ctypes.c_void_p(sums.data_ptr()),
        ctypes.c_void_p(keys.data_ptr()), int(keys.numel() // 4), ctypes.byref(n), bbox)
    _native.raise_for(rc, "sc_shard_mesh")
    return int(n.value), tuple(int(b) for b in bbox)


def shard_diameters(sums, keys, n_keys: int, shape, bbox, spacing: Sequence[float], shard: int,
                    nshards: int, sq4, stream=None) -> Coefficients:
    """Phase 2 of the slab-split shard (sc_shard_diameters): the summed partials,
    the gathered keys (first n_keys vertices of `keys`) and phase 1's bbox;
    shard `shard` of the pair grid, squared maxima into `sq4` (CUDA float64[4])
    for an all-reduce(MAX).  Counts, area and volume are complete."""
    sp = np.asarray(_check_spacing(spacing), dtype=np.float64)
    nz, ny, nx = (int(d) for d in shape)
    handle = _stream_handle(sums, stream)
    bb = (ctypes.c_int32 * 6)(*bbox)
    out = _native.ScCoeffs()
    rc = _native.load().sc_shard_diameters(
        ctypes.c_void_p(sums.data_ptr()), ctypes.c_void_p(keys.data_ptr()), int(n_keys),
        nx, ny, nz, bb, sp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
        ctypes.c_void_p(handle), int(shard), int(nshards), ctypes.c_void_p(sq4.data_ptr()),
        ctypes.byref(out))
    _native.raise_for(rc, "sc_shard_diameters")
    return _from_struct(out)


def calculate_coefficients_batch(masks: Sequence, spacings: Sequence[Sequence[float]],
                                 device: int = 0,
                                 devices: Optional[Sequence[int]] = None) -> List[Coefficients]:
    """C4: many host ROIs in one C call -- on `device`, or fanned out over
    `devices` inside the library (sc_calculate_coefficients_batch_multi: LPT
    placement, one host thread per device); records come back in input order."""
    bufs, dims = [], []
    for m in masks:
        data, d = _as_mask(m)
        bufs.append(data)
        dims.extend(d)
    sp = _check_spacings(spacings, len(bufs))
    n = len(bufs)
    ptrs = (ctypes.POINTER(ctypes.c_uint8) * n)(
        *[b.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)) for b in bufs])
    dims_arr = np.asarray(dims, dtype=np.int64)
    outs = (_native.ScCoeffs * n)()
    if devices is not None:
        devs = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
        rc = _native.load().sc_calculate_coefficients_batch_multi(
            ptrs, dims_arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
            sp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n, devs, len(devices), outs)
        _native.raise_for(rc, "sc_calculate_coefficients_batch_multi")
        return _from_structs(outs)
    rc = _native.load().sc_calculate_coefficients_batch(
        ptrs, dims_arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        sp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n, int(device), outs)
    _native.raise_for(rc, "sc_calculate_coefficients_batch")
    return _from_structs(outs)


def calculate_coefficients_device_batch(masks: Sequence, spacings: Sequence[Sequence[float]],
                                        stream=None) -> List[Coefficients]:
    """Many device-resident masks (CUDA uint8 tensors (nz, ny, nx) on the
    current device) in one pipelined C call, ordered after prior work on
    `stream` (a torch.cuda.Stream) and before later work on it."""
    n = len(masks)
    ptrs = (ctypes.c_void_p * n)(*[m.data_ptr() for m in masks])
    dims = np.asarray([(int(m.shape[2]), int(m.shape[1]), int(m.shape[0])) for m in masks],
                      dtype=np.int64).reshape(-1)
    sp = _check_spacings(spacings, n)
    for m in masks:
        if not m.is_contiguous():
            raise ValueError("device masks must be contiguous")
    outs = (_native.ScCoeffs * n)()
    handle = _stream_handle(masks[0], stream) if n else 0
    rc = _native.load().sc_calculate_coefficients_device_batch(
        ptrs, dims.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        sp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), n, ctypes.c_void_p(handle), outs)
    _native.raise_for(rc, "sc_calculate_coefficients_device_batch")
    return _from_structs(outs)


def _as_coord_arrays(xs, ys, zs):
    """features.py:195-202."""
    arrs = tuple(np.ascontiguousarray(a, dtype=np.float64) for a in (xs, ys, zs))
    n = arrs[0].shape[0]
    if n == 0:
        raise NoVertices("diameters need at least one vertex")
    if arrs[1].shape[0] != n or arrs[2].shape[0] != n:
        raise ValueError("coordinate arrays must have equal length")
    return arrs


def diameters(xs, ys, zs, device: int = 0) -> Tuple[float, float, float, float]:
    """(max_3d, xy, xz, yz) in mm, bit-exact with the reference (features.py:205-213)."""
    xs, ys, zs = _as_coord_arrays(xs, ys, zs)
    out = np.zeros(4, dtype=np.float64)
    dp = ctypes.POINTER(ctypes.c_double)
    rc = _native.load().sc_diameters(xs.ctypes.data_as(dp), ys.ctypes.data_as(dp),
                                     zs.ctypes.data_as(dp), xs.shape[0], int(device),
                                     out.ctypes.data_as(dp))
    _native.raise_for(rc, "sc_diameters")
    return tuple(float(v) for v in out)


def diameters_parallel(xs, ys, zs, workers: Optional[int] = None,
                       device: int = 0) -> Tuple[float, float, float, float]:
    """Reference signature (features.py:216-221); the GPU kernel is the only path."""
    return diameters(xs, ys, zs, device=device)


def mesh_vertices(mask, device: int = 0) -> np.ndarray:
    """(V, 3) int32 doubled lattice coordinates of the marching-cubes vertices
    (coordinate = key / 2 * spacing, mesh.py:182-195); order unspecified."""
    data, (nx, ny, nz) = _as_mask(mask)
    lib = _native.load()
    n = ctypes.c_int64()
    cap = 1 << 16
    while True:
        buf = np.empty((cap, 3), dtype=np.int32)
        rc = lib.sc_mesh_vertices(data.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), nx, ny,
                                  nz, int(device),
                                  buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), cap,
                                  ctypes.byref(n))
        _native.raise_for(rc, "sc_mesh_vertices")
        if n.value <= cap:
            return buf[: n.value].copy()
        cap = n.value


def extract_features(vol: MaskVolume, selection=None,
                     device: int = 0) -> Tuple[ShapeFeatures, StageTimings]:
    """features.py:224-265 on the B200.  Returns (ShapeFeatures, StageTimings);
    mesh_ms / diameters_ms are CUDA-event stage times, total_ms wall time."""
    t0 = now_ms()
    c = calculate_coefficients(vol.as_3d(), vol.spacing, device=device)
    t1 = now_ms()
    feats = ShapeFeatures(c.mesh_volume, c.surface_area, c.max_3d_diameter,
                          c.max_2d_diameter_xy, c.max_2d_diameter_xz, c.max_2d_diameter_yz,
                          c.vertex_count)
    total = max(t1 - t0, c.mesh_ms + c.diameters_ms)
    return feats, StageTimings(file_read_ms=0.0, mesh_ms=c.mesh_ms,
                               diameters_ms=c.diameters_ms, total_ms=total)
