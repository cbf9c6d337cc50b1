"""paper_2510_02894_b200: B200-native shape coefficients (PyRadiomics-cuda hot path).

Public API mirrors the reference `shapecore` package
(/root/reference/pkg/src/shapecore/__init__.py) for the hot path:
`extract_features`, `ShapeFeatures`, `FEATURE_KEYS`, `diameters`,
`diameters_parallel`, `MaskVolume`, `attach_spacing`, `StageTimings` and the
error classes, plus north_star's `calculate_coefficients(mask, spacing)`.
All compute runs in libshapecore_b200.so (sm_100a CUDA); importing this
package does not touch the GPU, calling it does.
"""

from .errors import (
    DeviceError,
    EmptyRoi,
    NonPositiveSpacing,
    NoVertices,
    ShapeCoreError,
    ShapeExceedsBounds,
)
from .features import (
    FEATURE_KEYS,
    Coefficients,
    ShapeFeatures,
    calculate_coefficients,
    calculate_coefficients_batch,
    calculate_coefficients_device,
    calculate_coefficients_device_batch,
    calculate_coefficients_shard,
    diameters,
    diameters_parallel,
    extract_features,
    mesh_vertices,
    shard_diameters,
    shard_exchange_sizes,
    shard_mesh,
)
from .mesh import (
    TriangleMesh,
    marching_cubes,
    mesh_dump,
    mesh_volume,
    signed_mesh_volume,
    surface_area,
    write_off,
    write_stl,
)
from .npy import (coefficients_from_npy, coefficients_from_npy_batch, coefficients_from_payloads,
                  load_npy, parse_npy_header)
from .pipeline import BenchRecord, bench_run, emit_tsv, parse_tsv, render_tsv, run_pipeline
from .synth import synth_mask
from .timing import StageTimings
from .volume import MaskVolume, attach_spacing

__version__ = "0.1.0"

__all__ = [
    "FEATURE_KEYS", "Coefficients", "DeviceError", "EmptyRoi", "MaskVolume", "NoVertices",
    "NonPositiveSpacing", "ShapeCoreError", "ShapeExceedsBounds", "ShapeFeatures",
    "StageTimings", "attach_spacing", "calculate_coefficients", "calculate_coefficients_batch",
    "calculate_coefficients_device", "calculate_coefficients_device_batch",
    "calculate_coefficients_shard", "diameters", "shard_diameters", "shard_exchange_sizes",
    "shard_mesh",
    "diameters_parallel", "extract_features", "mesh_vertices", "synth_mask",
    "coefficients_from_npy", "coefficients_from_npy_batch", "coefficients_from_payloads",
    "load_npy", "parse_npy_header", "BenchRecord", "bench_run",
    "emit_tsv", "parse_tsv", "render_tsv", "run_pipeline", "TriangleMesh", "marching_cubes",
    "mesh_dump", "mesh_volume", "signed_mesh_volume", "surface_area", "write_off", "write_stl",
]
