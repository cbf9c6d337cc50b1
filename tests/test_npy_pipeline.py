"""NPY loading, run_pipeline / bench TSV surface (8f #2) and the
in-process binding (8f #3).  CPU tests pin the host-side parsing against the
reference (when /root/reference is present); GPU tests pin the device
binarization and the full file -> coefficients path."""

import os
import sys

import numpy as np
import pytest

from conftest import REL_TOL, rel_err
from paper_2510_02894_b200 import errors, npy, pipeline

REF_SRC = "/tmp/refpkg/src"


def _ref():
    if not os.path.isdir("/root/reference"):
        pytest.skip("reference checkout not present")
    if not os.path.isdir(REF_SRC):
        import shutil

        shutil.copytree("/root/reference/pkg", "/tmp/refpkg")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import shapecore

    return shapecore


DTYPES = [np.bool_, np.uint8, np.int16, np.int32, np.int64, np.float32, np.float64]


def _write_cases(tmp_path, rng):
    files = []
    for i, dt in enumerate(DTYPES):
        for fortran in (False, True):
            arr = rng.integers(0, 4, size=(7, 9, 11)).astype(dt)
            if fortran:
                arr = np.asfortranarray(arr)
            p = tmp_path / f"m{i}_{int(fortran)}.npy"
            np.save(p, arr)
            files.append((p, arr))
    return files


def test_load_npy_matches_reference(tmp_path):
    sc = _ref()
    rng = np.random.default_rng(4)
    for p, arr in _write_cases(tmp_path, rng):
        for label in (None, 0, 2, 3):
            if arr.dtype == np.bool_ and label not in (None, 0):
                continue
            mine = npy.load_npy(p, label)
            ref = sc.load_npy(str(p), binarize_label=label)
            assert mine.dims == ref.dims
            assert np.array_equal(mine.data, ref.data), (p.name, label)


@pytest.mark.parametrize("content,exc", [
    (b"NOTNPY", errors.MalformedHeader),
    (b"\x93NUMPY\x03\x00", errors.MalformedHeader),
    (b"\x93NUMPY\x01\x00\x10\x00{'descr': '<i2'", errors.MalformedHeader),
])
def test_header_errors_match_reference(tmp_path, content, exc):
    p = tmp_path / "bad.npy"
    p.write_bytes(content)
    with pytest.raises(exc):
        npy.load_npy(p)
    if os.path.isdir("/root/reference"):
        sc = _ref()
        with pytest.raises(getattr(sc, exc.__name__)):
            sc.load_npy(str(p))


def test_dtype_shape_payload_errors(tmp_path):
    np.save(tmp_path / "c.npy", np.zeros((3, 3, 3), np.complex64))
    with pytest.raises(errors.UnsupportedDtype):
        npy.load_npy(tmp_path / "c.npy")
    np.save(tmp_path / "d.npy", np.zeros((3, 3), np.uint8))
    with pytest.raises(errors.NotThreeDimensional):
        npy.load_npy(tmp_path / "d.npy")
    np.save(tmp_path / "e.npy", np.zeros((4, 4, 4), np.int32))
    raw = (tmp_path / "e.npy").read_bytes()
    (tmp_path / "e.npy").write_bytes(raw[:-10])
    with pytest.raises(errors.TruncatedPayload):
        npy.load_npy(tmp_path / "e.npy")
    with pytest.raises(errors.IoFailure):
        npy.load_npy(tmp_path / "missing.npy")


def test_tsv_roundtrip_and_reference_compat(tmp_path):
    recs = [pipeline.BenchRecord("a", 100, 6, "b200", 0, 0.1234, 1.5, 2.25, 4.0),
            pipeline.BenchRecord("b", 200, 1248, "b200", 1, 0.5, 0.25, 0.125, 1.0)]
    p1 = tmp_path / "r1.tsv"
    pipeline.emit_tsv(recs, str(p1))
    back = pipeline.parse_tsv(str(p1))
    p2 = tmp_path / "r2.tsv"
    pipeline.emit_tsv(back, str(p2))
    assert p1.read_bytes() == p2.read_bytes()
    if os.path.isdir("/root/reference"):
        sc = _ref()
        ref_recs = sc.parse_tsv(str(p1))  # the reference reads our TSV
        p3 = tmp_path / "r3.tsv"
        sc.emit_tsv(ref_recs, str(p3))
        assert p3.read_bytes() == p1.read_bytes()  # ... and writes it back identically
    base = [pipeline.BenchRecord("a", 100, 6, "sequential", 0, 0.1, 30.0, 70.0, 110.0)]
    rows = pipeline.speedup_over_reference(back, base)
    assert len(rows) == 1 and rows[0].comp_speedup == pytest.approx(100.0 / 3.75)


def test_binding_input_errors_without_gpu():
    from paper_2510_02894_b200 import binding

    with pytest.raises(binding.InputError):
        binding.execute(np.zeros((3, 3), np.uint8))
    with pytest.raises(binding.InputError):
        binding.dump_arrays(np.zeros((2, 2)), np.zeros((2, 2, 2)), "/tmp")


# ------------------------------------------------------------------ GPU part
@pytest.mark.gpu
def test_device_binarization_all_dtypes(tmp_path, cuda_device):
    import paper_2510_02894_b200 as sc

    rng = np.random.default_rng(5)
    base = sc.synth_mask("ellipsoid", (21, 19, 17), semi_axes=(8, 7, 6)).astype(np.int64)
    base = base * rng.integers(1, 4, size=base.shape)  # labels 1..3 inside the shape
    for dt in DTYPES:
        for fortran in (False, True):
            arr = base.astype(dt)
            if fortran:
                arr = np.asfortranarray(arr)
            p = tmp_path / f"m_{np.dtype(dt).name}_{int(fortran)}.npy"
            np.save(p, arr)
            for label in ((None,) if dt == np.bool_ else (None, 2)):
                got, _ = npy.coefficients_from_npy(p, (0.8, 0.9, 1.1), label=label)
                host = npy.load_npy(p, label)
                want = sc.calculate_coefficients(host.as_3d(), (0.8, 0.9, 1.1))
                assert got.to_dict() == want.to_dict(), (p.name, label)
                assert got.triangle_count == want.triangle_count


@pytest.mark.gpu
def test_run_pipeline_and_bench_run(tmp_path, golden, oracle_mod, cuda_device):
    import paper_2510_02894_b200 as sc

    ds = tmp_path / "ds"
    ds.mkdir()
    vox = sc.synth_mask("box", (3, 3, 3), lo=(1, 1, 1), hi=(1, 1, 1))
    np.save(ds / "a.npy", vox)
    np.save(ds / "b.npy", sc.synth_mask("sphere", (24, 24, 24), radius=8).astype(np.int16) * 5)
    np.save(ds / "c_empty.npy", np.zeros((4, 4, 4), np.uint8))
    feats, t, sel = pipeline.run_pipeline(str(ds / "b.npy"), (1.0, 1.0, 1.0))
    assert feats.to_dict()["VertexCount"] == 1248  # README record (pkg/README.md:33-37)
    assert feats.max_3d_diameter == 16.792855623746664
    assert t.total_ms >= t.mesh_ms + t.diameters_ms and t.file_read_ms > 0
    assert sel.resolved == "b200"
    with pytest.raises(errors.EmptyRoi):
        pipeline.run_pipeline(str(ds / "c_empty.npy"))
    recs = pipeline.bench_run(str(ds), repeats=2, warmups=1)
    assert [r.case_id for r in recs] == ["a", "a", "b", "b", "c_empty"]
    assert recs[-1].error and recs[-1].total_ms == 0.0
    assert recs[0].vertex_count == 6 and recs[2].vertex_count == 1248


@pytest.mark.gpu
def test_binding_execute(tmp_path, golden, golden_arrays, cuda_device):
    from paper_2510_02894_b200 import binding

    case = golden["cases"][3]  # README sphere
    arr = golden_arrays[case["mask_key"]]
    rec = binding.execute(arr, case["spacing"])
    assert tuple(rec) == tuple(case["features"]) and rec == case["features"] | {
        "MeshVolume": rec["MeshVolume"], "SurfaceArea": rec["SurfaceArea"]}
    assert rel_err(rec["MeshVolume"], case["features"]["MeshVolume"]) <= REL_TOL
    img, msk = binding.dump_arrays(arr.astype(np.float32), arr, tmp_path)
    assert binding.execute(msk, case["spacing"])["VertexCount"] == case["features"]["VertexCount"]
    with pytest.raises(binding.EmptyRoi):
        binding.execute(np.zeros((4, 4, 4), np.uint8))
    (tmp_path / "bad.npy").write_bytes(b"garbage")
    with pytest.raises(binding.InputError):
        binding.execute(str(tmp_path / "bad.npy"))


@pytest.mark.gpu
def test_raw_payload_crop_chunks_fortran_labels(cuda_device):
    """SURVEY 8f #1 / VERDICT r01: typed payloads through the host slab crop,
    the chunked pinned staging (slabs of several 4 MB chunks), the chunk-wise
    binarize and the tiled Fortran transpose -- single entry, raw batch entry,
    pageable and pinned payloads, crop on and off -- all equal the uint8 host
    path on the reference-binarized mask (volume.py:173-177)."""
    import torch

    import paper_2510_02894_b200 as sc
    from paper_2510_02894_b200 import _native

    rng = np.random.default_rng(17)
    shapes = [(40, 96, 160), (37, 61, 83), (60, 256, 256)]  # (nz, ny, nx); x % 32 != 0 too
    cases = []
    for si, (nz, ny, nx) in enumerate(shapes):
        lab = np.zeros((nz, ny, nx), np.int64)
        for _ in range(6):
            c = rng.uniform([6, 6, 6], [nz - 6, ny - 6, nx - 6])
            r = rng.uniform(2, 5)
            zz, yy, xx = np.ogrid[:nz, :ny, :nx]
            lab[((zz - c[0]) ** 2 + (yy - c[1]) ** 2 + (xx - c[2]) ** 2) <= r * r] = \
                int(rng.integers(1, 4))
        for dt in DTYPES:
            base = (lab != 0) if dt == np.bool_ else lab.astype(dt)
            for fortran in (False, True):
                arr = np.asfortranarray(base) if fortran else np.ascontiguousarray(base)
                for label in ((None,) if dt == np.bool_ else (None, 2)):
                    cases.append((arr, label, (0.7, 0.8, 1.3)))
    want = []
    for arr, label, sp in cases:
        occ = (arr != 0) if label is None else (arr == arr.dtype.type(label))
        if not occ.any():
            want.append(None)
            continue
        want.append(sc.calculate_coefficients(np.ascontiguousarray(occ, np.uint8), sp).to_dict())
    keep = [(c, w) for c, w in zip(cases, want) if w is not None]
    payloads = [(a, lab) for (a, lab, _), _ in keep]
    sps = [sp for (_, _, sp), _ in keep]
    wants = [w for _, w in keep]
    for crop in (1, 0):
        with _native.thread_options(host_crop=crop):
            got = sc.coefficients_from_payloads(payloads, sps)
            assert [g.to_dict() for g in got] == wants, crop
    # pinned payloads take the direct 2-D copy path
    pinned = []
    for a, lab in payloads[:12]:
        t = torch.from_numpy(np.ascontiguousarray(a).view(np.uint8) if a.dtype == np.bool_
                             else np.ascontiguousarray(a)).pin_memory()
        pa = t.numpy().view(a.dtype) if a.dtype == np.bool_ else t.numpy()
        pinned.append((pa, lab))
    got = sc.coefficients_from_payloads(pinned, sps[:12])
    assert [g.to_dict() for g in got] == wants[:12]
    # an all-background payload is EmptyRoi, as the reference raises it
    with pytest.raises(errors.EmptyRoi):
        sc.coefficients_from_payloads([(np.zeros((8, 8, 8), np.int16), None)], [(1, 1, 1)])
