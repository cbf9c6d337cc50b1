"""Triangle mesh API on the B200.

Mirrors reference pkg/src/shapecore/mesh.py:28-252: `TriangleMesh`,
`marching_cubes(vol)`, the OFF/STL writers, and features.py:89-118
`surface_area` / `mesh_volume` / `signed_mesh_volume`.  The mesh comes from
`sc_marching_cubes` (canonical vertex numbering and triangle order, bit-exact
with the reference); the measures from `sc_mesh_measure` (the reference's
per-triangle arithmetic and pairwise fold, bit-exact).  The shape-coefficient
hot path never builds a mesh -- this is the export / inspection surface.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native
from .errors import EmptyRoi, IoFailure
from .volume import MaskVolume, _check_spacing


@dataclass(frozen=True)
class TriangleMesh:
    """Deduplicated surface in mm: xs/ys/zs per vertex, (n, 3) int32 triangles."""

    xs: np.ndarray
    ys: np.ndarray
    zs: np.ndarray
    triangles: np.ndarray

    def __post_init__(self):
        for arr in (self.xs, self.ys, self.zs, self.triangles):
            arr.flags.writeable = False

    @property
    def vertex_count(self) -> int:
        return int(self.xs.shape[0])

    @property
    def triangle_count(self) -> int:
        return int(self.triangles.shape[0])


def marching_cubes(vol: MaskVolume, device: int = 0) -> TriangleMesh:
    """mesh.py:68-91 on the GPU; raises EmptyRoi for an all-background mask."""
    data = np.ascontiguousarray(vol.data, dtype=np.uint8)
    nx, ny, nz = vol.dims
    sp = np.asarray(_check_spacing(vol.spacing), dtype=np.float64)
    lib = _native.load()
    u8 = data.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    dp = ctypes.POINTER(ctypes.c_double)
    nv, nt = ctypes.c_int64(), ctypes.c_int64()
    rc = lib.sc_marching_cubes(u8, nx, ny, nz, sp.ctypes.data_as(dp), int(device), None, None,
                               None, None, 0, 0, ctypes.byref(nv), ctypes.byref(nt))
    _native.raise_for(rc, "sc_marching_cubes")
    xs, ys, zs = (np.empty(nv.value, np.float64) for _ in range(3))
    tris = np.empty((nt.value, 3), np.int32)
    rc = lib.sc_marching_cubes(u8, nx, ny, nz, sp.ctypes.data_as(dp), int(device),
                               xs.ctypes.data_as(dp), ys.ctypes.data_as(dp),
                               zs.ctypes.data_as(dp),
                               tris.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), nv.value,
                               nt.value, ctypes.byref(nv), ctypes.byref(nt))
    _native.raise_for(rc, "sc_marching_cubes")
    return TriangleMesh(xs=xs, ys=ys, zs=zs, triangles=tris)


def _measure(mesh: TriangleMesh, device: int = 0):
    xs, ys, zs = (np.ascontiguousarray(a, dtype=np.float64) for a in (mesh.xs, mesh.ys, mesh.zs))
    tris = np.ascontiguousarray(mesh.triangles, dtype=np.int32).reshape(-1, 3)
    out = np.zeros(3)
    dp = ctypes.POINTER(ctypes.c_double)
    rc = _native.load().sc_mesh_measure(xs.ctypes.data_as(dp), ys.ctypes.data_as(dp),
                                        zs.ctypes.data_as(dp), xs.shape[0],
                                        tris.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                        tris.shape[0], int(device), out.ctypes.data_as(dp))
    _native.raise_for(rc, "sc_mesh_measure")
    return out


def surface_area(mesh: TriangleMesh) -> float:
    """features.py:89-96, bit-exact; 0.0 for an empty mesh."""
    return float(_measure(mesh)[0])


def signed_mesh_volume(mesh: TriangleMesh) -> float:
    """features.py:113-118, bit-exact."""
    return float(_measure(mesh)[1])


def mesh_volume(mesh: TriangleMesh) -> float:
    """features.py:99-110, bit-exact (abs applied once at the end)."""
    return float(_measure(mesh)[2])


def write_off(mesh: TriangleMesh, path) -> None:
    """ASCII OFF dump (mesh.py:202-213 format: repr floats)."""
    try:
        with Path(path).open("w", encoding="ascii") as fh:
            fh.write("OFF\n")
            fh.write(f"{mesh.vertex_count} {mesh.triangle_count} 0\n")
            for x, y, z in zip(mesh.xs.tolist(), mesh.ys.tolist(), mesh.zs.tolist()):
                fh.write(f"{x!r} {y!r} {z!r}\n")
            for a, b, c in mesh.triangles.tolist():
                fh.write(f"3 {a} {b} {c}\n")
    except OSError as exc:
        raise IoFailure(f"cannot write {path}: {exc}") from exc


def write_stl(mesh: TriangleMesh, path) -> None:
    """Binary STL dump (mesh.py:216-241 layout: 80-byte header, count, records)."""
    t = mesh.triangles
    corners = [np.column_stack((mesh.xs[t[:, k]], mesh.ys[t[:, k]], mesh.zs[t[:, k]]))
               for k in range(3)]
    normals = np.cross(corners[1] - corners[0], corners[2] - corners[0])
    lengths = np.linalg.norm(normals, axis=1)
    nz = lengths > 0
    normals[nz] /= lengths[nz, None]
    rec = np.empty(mesh.triangle_count,
                   dtype=[("n", "<f4", 3), ("v", "<f4", (3, 3)), ("attr", "<u2")])
    rec["n"] = normals
    for k in range(3):
        rec["v"][:, k, :] = corners[k]
    rec["attr"] = 0
    try:
        with Path(path).open("wb") as fh:
            fh.write(b"\0" * 80)
            fh.write(struct.pack("<I", mesh.triangle_count))
            fh.write(rec.tobytes())
    except OSError as exc:
        raise IoFailure(f"cannot write {path}: {exc}") from exc


def mesh_dump(mesh: TriangleMesh, path) -> None:
    """OFF or STL by extension (mesh.py:244-252)."""
    suffix = Path(path).suffix.lower()
    if suffix == ".off":
        write_off(mesh, path)
    elif suffix == ".stl":
        write_stl(mesh, path)
    else:
        raise IoFailure(f"mesh dump wants a .off or .stl path, got {path}")


__all__ = ["TriangleMesh", "marching_cubes", "surface_area", "mesh_volume",
           "signed_mesh_volume", "write_off", "write_stl", "mesh_dump", "EmptyRoi"]
