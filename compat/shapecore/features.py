"""shapecore.features on the B200 (reference features.py:27-265).

FEATURE_KEYS / ShapeFeatures / extract_features / diameters[_parallel] are the
B200 package's; surface_area / mesh_volume / signed_mesh_volume measure an
arbitrary TriangleMesh on the GPU with the reference's arithmetic
(sc_mesh_measure).  pairwise_sum is the reference's deterministic fold
(features.py:63-80), a host helper its tests call directly.
"""

import numpy as np

from paper_2510_02894_b200.features import (
    FEATURE_KEYS,
    ShapeFeatures,
    calculate_coefficients,
    diameters,
    diameters_parallel,
    extract_features,
)
from paper_2510_02894_b200.mesh import mesh_volume, signed_mesh_volume, surface_area


def pairwise_sum(values) -> float:
    """Zero-pad to the next power of two, then fold halves (a[:h] + a[h:])
    until one element is left: the summation tree depends only on the count."""
    v = np.asarray(values, dtype=np.float64).reshape(-1)
    if v.size == 0:
        return 0.0
    buf = np.zeros(1 << (v.size - 1).bit_length(), dtype=np.float64)
    buf[: v.size] = v
    while buf.size > 1:
        h = buf.size // 2
        buf = buf[:h] + buf[h:]
    return float(buf[0])


__all__ = ["FEATURE_KEYS", "ShapeFeatures", "calculate_coefficients", "diameters",
           "diameters_parallel", "extract_features", "mesh_volume", "pairwise_sum",
           "signed_mesh_volume", "surface_area"]
