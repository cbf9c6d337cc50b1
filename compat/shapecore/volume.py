"""shapecore.volume: the MaskVolume input record (B200 package) plus the
reference's synthetic-mask generator returning a MaskVolume
(volume.py:220-295) and an NPY v1.0 |u1 writer (volume.py:187-211)."""

import numpy as np

from paper_2510_02894_b200 import synth as _synth
from paper_2510_02894_b200.errors import IoFailure
from paper_2510_02894_b200.npy import load_npy
from paper_2510_02894_b200.volume import MaskVolume, attach_spacing


def synth_mask(kind, dims, *, radius=None, semi_axes=None, center=None, lo=None, hi=None,
               spacing=(1.0, 1.0, 1.0)) -> MaskVolume:
    """Deterministic sphere / ellipsoid / box mask as a MaskVolume."""
    arr = _synth.synth_mask(kind, dims, radius=radius, semi_axes=semi_axes, center=center,
                            lo=lo, hi=hi)
    nx, ny, nz = (int(d) for d in dims)
    return MaskVolume(dims=(nx, ny, nz), spacing=tuple(float(s) for s in spacing),
                      data=arr.reshape(-1))


def save_npy(vol: MaskVolume, path) -> None:
    """Version-1.0 NPY of 1-byte unsigned ints, shape (nz, ny, nx)."""
    try:
        with open(path, "wb") as fh:
            np.lib.format.write_array(fh, np.ascontiguousarray(vol.as_3d(), dtype=np.uint8),
                                      version=(1, 0), allow_pickle=False)
    except OSError as exc:
        raise IoFailure(f"cannot write {path!r}: {exc}") from exc


__all__ = ["MaskVolume", "attach_spacing", "load_npy", "save_npy", "synth_mask"]
