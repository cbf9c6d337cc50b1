"""ctypes binding of libshapecore_b200.so (the C ABI in include/shapecore_b200.h).

This is the thin layer north_star places in `pkg/binding`: plain pointers and
sizes cross the boundary, no torch types.  The library is built in-tree by
`__graft_entry__.build()` (nvcc, sm_100a).  There is NO fallback: if the .so is
missing or no CUDA device is usable, every compute call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# (SC_LIB: an alternative build of the same library, for A/B measurements)
LIB_PATH = os.environ.get("SC_LIB") or os.path.join(_HERE, "libshapecore_b200.so")

SC_OK = 0
SC_ERR_INPUT = 2
SC_ERR_EMPTY_ROI = 3
SC_ERR_NO_VERTICES = 4
SC_ERR_CUDA = -1
SC_ERR_NOMEM = -2

EXPORTED = (
    "sc_calculate_coefficients",
    "sc_calculate_coefficients_device",
    "sc_calculate_coefficients_shard",
    "sc_shard_exchange_sizes",
    "sc_shard_mesh",
    "sc_shard_diameters",
    "sc_calculate_coefficients_raw",
    "sc_calculate_coefficients_raw_batch",
    "sc_calculate_coefficients_batch",
    "sc_calculate_coefficients_device_batch",
    "sc_calculate_coefficients_batch_multi",
    "sc_diameters",
    "sc_mesh_vertices",
    "sc_marching_cubes",
    "sc_mesh_measure",
    "sc_last_kernel_times",
    "sc_last_diagnostics",
    "sc_set_option",
    "sc_set_thread_option",
    "sc_clear_thread_options",
    "sc_launch_count",
    "sc_probe_fp32_peak",
    "sc_occupied_slab",
    "sc_last_error",
    "sc_abi_version",
    "sc_device_count",
)


class ScRawMask(ctypes.Structure):
    """Mirror of `sc_raw_mask` (include/shapecore_b200.h)."""

    _fields_ = [
        ("data", ctypes.c_void_p),
        ("dtype", ctypes.c_int),
        ("fortran_order", ctypes.c_int),
        ("has_label", ctypes.c_int),
        ("label_int", ctypes.c_int64),
        ("label_float", ctypes.c_double),
        ("shape", ctypes.c_int64 * 3),
    ]


class ScCoeffs(ctypes.Structure):
    """Mirror of `sc_coeffs` (include/shapecore_b200.h)."""

    _fields_ = [
        ("mesh_volume", ctypes.c_double),
        ("surface_area", ctypes.c_double),
        ("max_3d_diameter", ctypes.c_double),
        ("max_2d_diameter_xy", ctypes.c_double),
        ("max_2d_diameter_xz", ctypes.c_double),
        ("max_2d_diameter_yz", ctypes.c_double),
        ("vertex_count", ctypes.c_int64),
        ("triangle_count", ctypes.c_int64),
        ("active_cubes", ctypes.c_int64),
        ("h2d_ms", ctypes.c_double),
        ("mesh_ms", ctypes.c_double),
        ("diameters_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double),
        ("h2d_bytes", ctypes.c_int64),
        ("host_scan_ms", ctypes.c_double),
    ]


_lib = None
_lock = threading.Lock()


def load():
    """Load the native library (raises OSError if it was not built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise OSError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (nvcc, sm_100a).  There is no CPU fallback."
            )
        L = ctypes.CDLL(LIB_PATH)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        dp = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        cp = ctypes.POINTER(ScCoeffs)
        L.sc_calculate_coefficients.argtypes = [u8p, i64, i64, i64, dp, ctypes.c_int, cp]
        L.sc_calculate_coefficients_device.argtypes = [ctypes.c_void_p, i64, i64, i64, dp,
                                                       ctypes.c_void_p, cp]
        L.sc_calculate_coefficients_shard.argtypes = [ctypes.c_void_p, i64, i64, i64, dp,
                                                      ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                                      ctypes.c_void_p, cp]
        i64p = ctypes.POINTER(i64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        ab = bool(os.environ.get("SC_LIB"))  # an older A/B build may lack newer entries
        if not ab or hasattr(L, "sc_shard_mesh"):
            L.sc_shard_exchange_sizes.argtypes = [i64, i64, i64, i64p, i64p]
            L.sc_shard_mesh.argtypes = [ctypes.c_void_p, i64, i64, i64, dp, ctypes.c_void_p,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                        ctypes.c_void_p,
                                        i64, i64p, i32p]
            L.sc_shard_diameters.argtypes = [ctypes.c_void_p, ctypes.c_void_p, i64, i64, i64,
                                             i64, i32p, dp, ctypes.c_void_p, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_void_p, cp]
        L.sc_calculate_coefficients_batch.argtypes = [ctypes.POINTER(u8p),
                                                      ctypes.POINTER(i64), dp, i64,
                                                      ctypes.c_int, cp]
        L.sc_calculate_coefficients_batch_multi.argtypes = [ctypes.POINTER(u8p),
                                                            ctypes.POINTER(i64), dp, i64,
                                                            ctypes.POINTER(ctypes.c_int),
                                                            ctypes.c_int, cp]
        L.sc_calculate_coefficients_device_batch.argtypes = [ctypes.POINTER(ctypes.c_void_p),
                                                             ctypes.POINTER(i64), dp, i64,
                                                             ctypes.c_void_p, cp]
        L.sc_calculate_coefficients_raw.argtypes = [ctypes.c_void_p, ctypes.c_int,
                                                    ctypes.POINTER(i64), ctypes.c_int,
                                                    ctypes.c_int, i64, ctypes.c_double, dp,
                                                    ctypes.c_int, cp]
        L.sc_calculate_coefficients_raw_batch.argtypes = [ctypes.POINTER(ScRawMask), dp, i64,
                                                          ctypes.c_int, cp]
        L.sc_diameters.argtypes = [dp, dp, dp, i64, ctypes.c_int, dp]
        L.sc_mesh_vertices.argtypes = [u8p, i64, i64, i64, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_int32), i64,
                                       ctypes.POINTER(i64)]
        L.sc_marching_cubes.argtypes = [u8p, i64, i64, i64, dp, ctypes.c_int, dp, dp, dp,
                                        ctypes.POINTER(ctypes.c_int32), i64, i64,
                                        ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.sc_mesh_measure.argtypes = [dp, dp, dp, i64, ctypes.POINTER(ctypes.c_int32), i64,
                                      ctypes.c_int, dp]
        L.sc_last_kernel_times.argtypes = [ctypes.c_int, dp, ctypes.c_int]
        L.sc_launch_count.restype = ctypes.c_uint64
        L.sc_last_diagnostics.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
        L.sc_set_option.argtypes = [ctypes.c_char_p, ctypes.c_int]
        L.sc_set_thread_option.argtypes = [ctypes.c_char_p, ctypes.c_int]
        L.sc_clear_thread_options.restype = None
        L.sc_probe_fp32_peak.argtypes = [ctypes.c_int, ctypes.c_int, dp]
        L.sc_occupied_slab.argtypes = [u8p, i64, i64, i64, ctypes.c_int, ctypes.POINTER(i64)]
        L.sc_last_error.restype = ctypes.c_char_p
        L.sc_abi_version.restype = ctypes.c_int
        L.sc_device_count.restype = ctypes.c_int
        for name in EXPORTED:
            if not hasattr(L, name) and not (ab and name.startswith("sc_shard_")):
                raise OSError(f"{LIB_PATH} does not export {name}")
        _lib = L
        return L


def last_error() -> str:
    msg = load().sc_last_error()
    return msg.decode() if msg else ""


def raise_for(rc: int, what: str = "") -> None:
    """Map C return codes onto the reference exception classes (errors.py)."""
    if rc == SC_OK:
        return
    from . import errors

    msg = last_error() or what
    if rc == SC_ERR_EMPTY_ROI:
        raise errors.EmptyRoi(msg)
    if rc == SC_ERR_NO_VERTICES:
        raise errors.NoVertices(msg)
    if rc == SC_ERR_INPUT:
        if "spacing" in msg:
            raise errors.NonPositiveSpacing(msg)
        raise ValueError(msg)
    raise errors.DeviceError(f"{what}: {msg} (code {rc})")


# Stage times of the last ROI: HBM pack, bbox + marching cubes, 3-D sort/boxes/
# filter, pass 1 (3-D + planar lists), exact re-check (both), planar prep
# (plane boxes / lower bounds / filter), host->device copy.
KERNEL_TIME_NAMES = ("pack_ms", "mc_ms", "prune_ms", "pass1_ms", "refine_ms", "planar_prep_ms",
                     "h2d_ms")


def last_kernel_times(device: int = 0) -> dict:
    """Per-kernel CUDA-event times (ms) of the last ROI on `device`."""
    buf = (ctypes.c_double * 7)()
    n = load().sc_last_kernel_times(int(device), buf, 7)
    if n < 0:
        raise_for(-n, "sc_last_kernel_times")
    return {k: buf[i] for i, k in enumerate(KERNEL_TIME_NAMES[:n])}


def launch_count() -> int:
    return int(load().sc_launch_count())


def probe_fp32_peak(device: int = 0, mode: int = 0) -> float:
    """Measured FP32 CUDA-core TFLOP/s (mode 0: FFMA2, mode 1: FFMA)."""
    out = ctypes.c_double()
    raise_for(load().sc_probe_fp32_peak(int(device), int(mode), ctypes.byref(out)),
              "sc_probe_fp32_peak")
    return out.value


DIAG_NAMES = ("work_units", "total_units", "refine_candidates", "planar_units",
              "planar_candidates", "planar_work_units", "work_subunits", "planar_work_subunits",
              "pass1_pairs", "pass1_planar_pairs")
PAIRS_PER_UNIT = 128 * 128


def last_diagnostics(device: int = 0) -> dict:
    buf = (ctypes.c_int64 * len(DIAG_NAMES))()
    n = load().sc_last_diagnostics(int(device), buf, len(DIAG_NAMES))
    if n < 0:
        raise_for(-n, "sc_last_diagnostics")
    return {k: int(buf[i]) for i, k in enumerate(DIAG_NAMES[:n])}


def set_option(name: str, value: int) -> None:
    """Process-wide option (calls already in flight keep their snapshot)."""
    raise_for(load().sc_set_option(name.encode(), int(value)), "sc_set_option")


class thread_options:
    """`with thread_options(prune=0, slots=8): ...` -- options for the calls
    made from this thread only (sc_set_thread_option); restored on exit."""

    def __init__(self, **opts):
        self.opts = opts

    def __enter__(self):
        for k, v in self.opts.items():
            raise_for(load().sc_set_thread_option(k.encode(), int(v)), "sc_set_thread_option")
        return self

    def __exit__(self, *exc):
        load().sc_clear_thread_options()


def occupied_slab(mask, threads: int = 0):
    """(z0, z1, y0, y1) occupied extent of a C-contiguous (nz, ny, nx) uint8
    mask via the library's host scan (no device needed); None if empty."""
    import numpy as np

    arr = np.ascontiguousarray(mask, dtype=np.uint8)
    nz, ny, nx = arr.shape
    out = (ctypes.c_int64 * 4)()
    rc = load().sc_occupied_slab(arr.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), nx, ny,
                                 nz, int(threads), out)
    if rc == 3:
        return None
    if rc != 0:
        raise ValueError(last_error())
    return tuple(int(v) for v in out)
