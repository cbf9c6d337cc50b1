"""Input record of the hot path: a binary voxel grid with physical spacing.

Mirror of reference `MaskVolume` (pkg/src/shapecore/volume.py:59-101): dims is
(nx, ny, nz); data is a flat uint8 array in C order with x fastest, i.e.
data[(iz * ny + iy) * nx + ix].  Any nonzero byte counts as occupied on the
B200 path (the reference only ever sees 0/1 data).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import Optional, Sequence, Tuple

import numpy as np

from .errors import NonPositiveSpacing


def _check_spacing(spacing: Sequence[float]) -> Tuple[float, float, float]:
    """volume.py:94-101: three finite components, each > 0."""
    vals = tuple(float(s) for s in spacing)
    if len(vals) != 3:
        raise NonPositiveSpacing(f"spacing needs 3 components, got {len(vals)}")
    for s in vals:
        if not (s > 0.0) or not math.isfinite(s):
            raise NonPositiveSpacing(f"spacing components must be finite and > 0, got {vals}")
    return vals


@dataclass(frozen=True)
class MaskVolume:
    dims: Tuple[int, int, int]
    spacing: Tuple[float, float, float]
    data: np.ndarray
    label: Optional[int] = None

    def __post_init__(self):
        nx, ny, nz = self.dims
        if min(nx, ny, nz) < 1:
            raise ValueError(f"dims must all be >= 1, got {self.dims}")
        if self.data.size != nx * ny * nz:
            raise ValueError(f"data length {self.data.size} != nx*ny*nz = {nx * ny * nz}")
        _check_spacing(self.spacing)
        self.data.flags.writeable = False

    @property
    def occupied_count(self) -> int:
        return int(np.count_nonzero(self.data))

    def as_3d(self) -> np.ndarray:
        nx, ny, nz = self.dims
        return self.data.reshape(nz, ny, nx)

    @classmethod
    def from_array(cls, arr: np.ndarray, spacing=(1.0, 1.0, 1.0)) -> "MaskVolume":
        """Wrap a (nz, ny, nx) array (nonzero = occupied) without binarizing."""
        if arr.ndim != 3:
            raise ValueError(f"mask array must be 3-D, got {arr.ndim}-D")
        nz, ny, nx = arr.shape
        data = np.ascontiguousarray(arr)
        if data.dtype != np.uint8:
            data = (data != 0).astype(np.uint8)
        return cls(dims=(nx, ny, nz), spacing=tuple(float(s) for s in spacing),
                   data=data.reshape(-1))


def attach_spacing(vol: MaskVolume, spacing: Sequence[float]) -> MaskVolume:
    """volume.py:215-217."""
    return replace(vol, spacing=_check_spacing(spacing))
