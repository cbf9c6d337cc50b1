"""`shapecore` compatibility package: the reference's import surface over the
B200 path.

The reference's callers import `shapecore` (/root/reference/pkg/src/shapecore,
__init__.py:9-57).  With `compat/` on sys.path ahead of (or instead of) the
reference, `import shapecore` resolves here and every hot-path name --
extract_features, marching_cubes, surface_area, mesh_volume, diameters,
diameters_parallel, MaskVolume, ShapeFeatures, TriangleMesh, the error
classes -- is the B200 implementation (paper_2510_02894_b200, the C ABI in
libshapecore_b200.so).  There is one backend: resolve_backend() accepts the
reference's names and returns a record for signature compatibility; nothing
dispatches on it and nothing falls back to the CPU.

Names outside the hot path that the reference's callers also use (synth_mask,
save_npy, pad_mask, pairwise_sum, the bench/TSV helpers) are thin host-side
mirrors.  tests/test_reference_suite.py runs the reference's own
test_features.py, test_mesh.py and test_acceptance.py against this package.
"""

from paper_2510_02894_b200.errors import (
    DeviceError,
    EmptyRoi,
    IoFailure,
    MalformedHeader,
    MissingBaseline,
    NoCasesFound,
    NonPositiveSpacing,
    NoRecords,
    NotThreeDimensional,
    NoVertices,
    ShapeCoreError,
    ShapeExceedsBounds,
    TruncatedPayload,
    UnsupportedDtype,
)
from paper_2510_02894_b200.timing import StageTimings

from .bench import BenchRecord, bench_run, emit_tsv, parse_tsv, render_tsv, speedup_table
from .dispatch import BackendSelection, hardware_worker_count, probe_parallel, resolve_backend, \
    run_pipeline
from .features import (
    ShapeFeatures,
    calculate_coefficients,
    diameters,
    diameters_parallel,
    extract_features,
    mesh_volume,
    surface_area,
)
from .mesh import TriangleMesh, marching_cubes, mesh_dump, write_off, write_stl
from .volume import MaskVolume, attach_spacing, load_npy, save_npy, synth_mask

__version__ = "1.0.0+b200"

__all__ = [
    "BackendSelection", "BenchRecord", "DeviceError", "EmptyRoi", "IoFailure", "MalformedHeader",
    "MaskVolume", "MissingBaseline", "NoCasesFound", "NonPositiveSpacing", "NoRecords",
    "NotThreeDimensional", "NoVertices", "ShapeCoreError", "ShapeExceedsBounds", "ShapeFeatures",
    "StageTimings", "TriangleMesh", "TruncatedPayload", "UnsupportedDtype", "attach_spacing",
    "bench_run", "calculate_coefficients", "diameters", "diameters_parallel", "emit_tsv",
    "extract_features", "hardware_worker_count", "load_npy", "marching_cubes", "mesh_dump",
    "mesh_volume", "parse_tsv", "probe_parallel", "render_tsv", "resolve_backend",
    "run_pipeline", "save_npy", "speedup_table", "surface_area", "synth_mask", "write_off",
    "write_stl",
]
