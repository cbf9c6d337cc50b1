"""CPU-side checks of the boundary: the C ABI library loads and exports every
entry point include/shapecore_b200.h declares, the ctypes record mirrors the C
struct, and the host-side argument handling mirrors the reference (no GPU
compute here)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def native():
    from paper_2510_02894_b200 import _native

    if not os.path.exists(_native.LIB_PATH):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2510_02894_b200", "csrc")],
                       check=True)
    return _native


def header_functions():
    src = open(os.path.join(ROOT, "include", "shapecore_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sc_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_header(native):
    lib = native.load()
    names = header_functions()
    assert "sc_calculate_coefficients" in names and len(names) >= 9
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(native.EXPORTED)
    assert lib.sc_abi_version() == 4


def test_nm_shows_c_symbols(native):
    out = subprocess.run(["nm", "-D", "--defined-only", native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    for name in header_functions():
        assert re.search(rf"\bT {name}$", out, flags=re.M), name


def test_struct_layout_matches_header(native):
    # 6 doubles, 3 int64, 4 doubles
    assert ctypes.sizeof(native.ScCoeffs) == 15 * 8
    src = open(os.path.join(ROOT, "include", "shapecore_b200.h")).read()
    body = src[src.index("typedef struct {"):src.index("} sc_coeffs;")]
    fields = re.findall(r"(double|int64_t)\s+(\w+);", body)
    assert [f for _, f in fields] == [f for f, _ in native.ScCoeffs._fields_]


def test_input_validation_without_gpu(native):
    lib = native.load()
    out = native.ScCoeffs()
    sp = (ctypes.c_double * 3)(1.0, 1.0, 1.0)
    buf = (ctypes.c_uint8 * 8)()
    rc = lib.sc_calculate_coefficients(buf, 0, 2, 2, sp, 0, ctypes.byref(out))
    assert rc == native.SC_ERR_INPUT and "dims" in native.last_error()
    bad = (ctypes.c_double * 3)(1.0, -1.0, 1.0)
    rc = lib.sc_calculate_coefficients(buf, 2, 2, 2, bad, 0, ctypes.byref(out))
    assert rc == native.SC_ERR_INPUT and "spacing" in native.last_error()
    dp = ctypes.POINTER(ctypes.c_double)
    out4 = (ctypes.c_double * 4)()
    rc = lib.sc_diameters(None, None, None, 0, 0, out4)
    assert rc == native.SC_ERR_NO_VERTICES


def test_error_mapping(native):
    import paper_2510_02894_b200 as sc

    with pytest.raises(sc.NonPositiveSpacing):
        sc.calculate_coefficients(np.ones((3, 3, 3), np.uint8), (0.0, 1.0, 1.0))
    with pytest.raises(sc.NoVertices):
        sc.diameters([], [], [])
    with pytest.raises(ValueError):
        sc.diameters([1.0, 2.0], [1.0], [1.0, 2.0])
    with pytest.raises(ValueError):
        sc.calculate_coefficients(np.ones((3, 3), np.uint8))


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback(native):
    """Without a device the product path fails loudly instead of computing."""
    import paper_2510_02894_b200 as sc

    with pytest.raises(sc.DeviceError):
        sc.calculate_coefficients(np.ones((3, 3, 3), np.uint8))
    with pytest.raises(sc.DeviceError):
        sc.diameters([0.0, 1.0], [0.0, 1.0], [0.0, 1.0])


def test_mask_volume_mirror():
    import paper_2510_02894_b200 as sc

    vol = sc.MaskVolume.from_array(np.ones((2, 3, 4), np.uint8), (1, 2, 3))
    assert vol.dims == (4, 3, 2) and vol.occupied_count == 24
    assert vol.as_3d().shape == (2, 3, 4)
    with pytest.raises(sc.NonPositiveSpacing):
        sc.attach_spacing(vol, (1, 0, 1))
    with pytest.raises(ValueError):
        sc.MaskVolume(dims=(2, 2, 2), spacing=(1, 1, 1), data=np.zeros(7, np.uint8))


def test_tables_header_matches_reference():
    ref = "/root/reference/pkg/src/shapecore/mc_tables.py"
    if not os.path.exists(ref):
        pytest.skip("reference checkout not present (GPU box)")
    import importlib.util

    spec = importlib.util.spec_from_file_location("ref_tables", ref)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    hdr = open(os.path.join(ROOT, "paper_2510_02894_b200", "csrc", "mc_tables.h")).read()
    rows = re.findall(r"\{([-0-9,]+)\},", hdr)
    table = np.array([[int(v) for v in r.split(",")] for r in rows])
    assert np.array_equal(table, mod.TRI_TABLE)
    for name in ("EDGE_AXIS", "EDGE_DX", "EDGE_DY", "EDGE_DZ"):
        vals = re.search(rf"SC_{name}\[12\] = \{{([-0-9,]+)\}}", hdr).group(1)
        assert [int(v) for v in vals.split(",")] == getattr(mod, name).tolist()


def test_occupied_slab_host_scan(native):
    """The host scan behind option host_crop (no device needed) finds the exact
    occupied z/y extent, with any thread count, odd row lengths included."""
    rng = np.random.default_rng(5)
    for trial in range(40):
        nz, ny, nx = (int(v) for v in rng.integers(1, 40, 3))
        if trial % 5 == 0:
            nx = int(rng.integers(100, 700))  # rows longer than one 32-byte step
        arr = np.zeros((nz, ny, nx), dtype=np.uint8)
        if trial % 7 == 0:
            for t in (1, 3):
                assert native.occupied_slab(arr, threads=t) is None
            continue
        k = int(rng.integers(1, 6))
        idx = (rng.integers(0, nz, k), rng.integers(0, ny, k), rng.integers(0, nx, k))
        arr[idx] = rng.integers(1, 256, k).astype(np.uint8)
        zs, ys = np.nonzero(arr.any(axis=2))
        want = (zs.min(), zs.max(), ys.min(), ys.max())
        for t in (1, 2, 7, 0):
            assert native.occupied_slab(arr, threads=t) == tuple(int(v) for v in want)
    big = np.zeros((600, 64, 512), dtype=np.uint8)  # noqa: E501
    big[300, 40, 511] = 1
    big[17, 3, 0] = 9
    assert native.occupied_slab(big, threads=8) == (17, 300, 3, 40)
