"""shapecore.mesh on the B200 (reference mesh.py:28-252): the canonical
TriangleMesh from sc_marching_cubes (bit-exact vertex numbering, coordinates
and triangle order) and the OFF / STL writers.  pad_mask is the reference's
host-side zero shell (mesh.py:55-65); the B200 path never materialises it."""

import numpy as np

from paper_2510_02894_b200.mesh import TriangleMesh, marching_cubes, mesh_dump, write_off, \
    write_stl

from .volume import MaskVolume


def pad_mask(vol: MaskVolume) -> MaskVolume:
    """One layer of background voxels on all six faces."""
    nx, ny, nz = vol.dims
    padded = np.zeros((nz + 2, ny + 2, nx + 2), dtype=np.uint8)
    padded[1:-1, 1:-1, 1:-1] = vol.as_3d()
    return MaskVolume(dims=(nx + 2, ny + 2, nz + 2), spacing=vol.spacing,
                      data=padded.reshape(-1), label=vol.label)


__all__ = ["TriangleMesh", "marching_cubes", "mesh_dump", "pad_mask", "write_off", "write_stl"]
