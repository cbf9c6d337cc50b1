"""GPU parity: the CUDA path (through the C ABI) against the reference.

Expected values come from tests/golden (frozen outputs of the reference,
tools/make_golden.py) and from the CPU oracle.  Bars (north_star):
  * bit-exact: vertex / triangle / active-cube counts, and -- because the
    diameter stage re-checks its candidates in the reference's own fp64
    arithmetic -- all four diameters;
  * relative error <= 1e-6 (REL_TOL) for surface area and mesh volume (the GPU
    sums exact integer histograms; the reference sums per-triangle floats).
"""

import hashlib
import math

import numpy as np
import pytest

from conftest import REL_TOL, rel_err

pytestmark = pytest.mark.gpu

DIAM_KEYS = ("Maximum3DDiameter", "Maximum2DDiameterXY", "Maximum2DDiameterXZ",
             "Maximum2DDiameterYZ")


def assert_matches(got, want_features, triangles, active, label=""):
    rec = got.to_dict()
    assert rec["VertexCount"] == want_features["VertexCount"], label
    assert got.triangle_count == triangles, label
    assert got.active_cubes == active, label
    for k in DIAM_KEYS:
        assert rec[k] == want_features[k], (label, k, rec[k], want_features[k])
    for k in ("MeshVolume", "SurfaceArea"):
        assert rel_err(rec[k], want_features[k]) <= REL_TOL, (label, k, rec[k], want_features[k])


def test_golden_small_cases(sc, golden, golden_arrays, cuda_device):
    worst = 0.0
    for case in golden["cases"]:
        arr = golden_arrays[case["mask_key"]]
        got = sc.calculate_coefficients(arr, case["spacing"], device=cuda_device)
        assert_matches(got, case["features"], case["triangle_count"], case["active_cubes"],
                       case["name"])
        for k in ("MeshVolume", "SurfaceArea"):
            worst = max(worst, rel_err(got.to_dict()[k], case["features"][k]))
    assert worst <= 1e-12  # in practice: only summation-order differences


def test_vertex_sets_match_reference(sc, golden, golden_arrays, cuda_device):
    n = 0
    for case in golden["cases"]:
        if "verts_key" not in case:
            continue
        sp = np.asarray(case["spacing"])
        keys = sc.mesh_vertices(golden_arrays[case["mask_key"]], device=cuda_device)
        got = keys.astype(np.float64) * 0.5 * sp  # same arithmetic as mesh.py:184-195
        want = golden_arrays[case["verts_key"]]
        assert got.shape == want.shape, case["name"]
        assert set(map(tuple, got.tolist())) == set(map(tuple, want.tolist())), case["name"]
        assert len(set(map(tuple, keys.tolist()))) == len(keys)  # deduplicated
        n += 1
    assert n >= 10


def test_clouds_bit_exact(sc, golden, golden_clouds, cuda_device):
    for c in golden["clouds"]:
        xs, ys, zs = golden_clouds[c["key"]]
        assert list(sc.diameters(xs, ys, zs, device=cuda_device)) == c["diameters"], c["key"]


def test_known_answers(sc, cuda_device):
    # pkg/tests/test_features.py:62-89, test_acceptance.py:20-39
    vox = sc.synth_mask("box", (3, 3, 3), lo=(1, 1, 1), hi=(1, 1, 1))
    c = sc.calculate_coefficients(vox, (1, 1, 1), device=cuda_device)
    assert c.vertex_count == 6 and c.triangle_count == 8
    assert abs(c.mesh_volume - 1 / 6) <= 1e-9 and abs(c.surface_area - math.sqrt(3)) <= 1e-9
    assert (c.max_3d_diameter, c.max_2d_diameter_xy, c.max_2d_diameter_xz,
            c.max_2d_diameter_yz) == (1.0, 1.0, 1.0, 1.0)
    assert sc.diameters([0.0, 3.0], [0.0, 4.0], [0.0, 0.0]) == (5.0, 5.0, 0.0, 0.0)
    assert sc.diameters([2.5], [2.5], [2.5]) == (0.0, 0.0, 0.0, 0.0)


def test_errors(sc, cuda_device):
    with pytest.raises(sc.EmptyRoi):
        sc.calculate_coefficients(np.zeros((4, 4, 4), np.uint8), device=cuda_device)
    with pytest.raises(sc.EmptyRoi):
        sc.calculate_coefficients(np.zeros((3, 5, 64), np.uint8), device=cuda_device)
    with pytest.raises(sc.NonPositiveSpacing):
        sc.calculate_coefficients(np.ones((3, 3, 3), np.uint8), (1.0, 0.0, 1.0))
    with pytest.raises(sc.NonPositiveSpacing):
        sc.calculate_coefficients(np.ones((3, 3, 3), np.uint8), (1.0, float("nan"), 1.0))
    with pytest.raises(sc.NoVertices):
        sc.diameters(np.zeros(0), np.zeros(0), np.zeros(0))


def test_aligned_and_generic_pack_paths_agree(sc, oracle_mod, cuda_device):
    """nx % 32 == 0 takes the 128-bit path; x offsets exercise word seams."""
    rng = np.random.default_rng(3)
    for nx in (32, 64, 96, 31, 33, 65):
        arr = (rng.random((9, 7, nx)) < 0.3).astype(np.uint8)
        arr[:, :, 0] = 1  # occupied voxels on the x faces and the word seams
        arr[:, :, -1] = 1
        want = oracle_mod.extract_features(arr, (1.0, 1.0, 1.0), threads=0)
        got = sc.calculate_coefficients(arr, (1.0, 1.0, 1.0), device=cuda_device)
        assert got.vertex_count == want["VertexCount"], nx
        assert got.triangle_count == want["triangle_count"], nx
        assert got.active_cubes == want["active_cubes"], nx
        for k in DIAM_KEYS:
            assert got.to_dict()[k] == want[k], (nx, k)
        for k in ("MeshVolume", "SurfaceArea"):
            assert rel_err(got.to_dict()[k], want[k]) <= REL_TOL


def test_nonbinary_values_count_as_occupied(sc, oracle_mod, cuda_device):
    arr = sc.synth_mask("sphere", (20, 20, 32), radius=6).astype(np.uint8) * 7
    a = sc.calculate_coefficients(arr, device=cuda_device)
    b = sc.calculate_coefficients((arr != 0).astype(np.uint8), device=cuda_device)
    assert a.to_dict() == b.to_dict()


def test_spacing_scaling_exact(sc, cuda_device):
    # pkg/tests/test_acceptance.py:102-116
    vol = sc.synth_mask("ellipsoid", (24, 22, 20), semi_axes=(8, 7, 6))
    f1 = sc.calculate_coefficients(vol, (1.0, 1.0, 1.0))
    f2 = sc.calculate_coefficients(vol, (2.0, 2.0, 2.0))
    assert f2.mesh_volume == 8.0 * f1.mesh_volume
    assert f2.surface_area == 4.0 * f1.surface_area
    assert f2.max_3d_diameter == 2.0 * f1.max_3d_diameter
    assert f2.max_2d_diameter_xy == 2.0 * f1.max_2d_diameter_xy
    assert f2.max_2d_diameter_xz == 2.0 * f1.max_2d_diameter_xz
    assert f2.max_2d_diameter_yz == 2.0 * f1.max_2d_diameter_yz


def test_axis_swap_permutes_planar(sc, cuda_device):
    # pkg/tests/test_features.py:173-190
    arr = sc.synth_mask("ellipsoid", (26, 22, 18), semi_axes=(9.0, 7.0, 5.5))
    f0 = sc.calculate_coefficients(arr, (1.0, 0.5, 2.0))
    f1 = sc.calculate_coefficients(np.ascontiguousarray(arr.transpose(0, 2, 1)), (0.5, 1.0, 2.0))
    assert f1.vertex_count == f0.vertex_count
    assert f1.max_2d_diameter_xy == f0.max_2d_diameter_xy
    assert f1.max_2d_diameter_xz == f0.max_2d_diameter_yz
    assert f1.max_2d_diameter_yz == f0.max_2d_diameter_xz


def test_extract_features_api(sc, cuda_device):
    vol = sc.MaskVolume.from_array(sc.synth_mask("sphere", (40, 40, 40), radius=15))
    feats, t = sc.extract_features(vol)
    assert tuple(feats.to_dict()) == sc.FEATURE_KEYS
    assert isinstance(feats.to_dict()["VertexCount"], int)
    assert t.total_ms >= t.mesh_ms + t.diameters_ms
    assert 28.0 <= feats.max_3d_diameter <= 32.0


def _big(sc, name):
    from paper_2510_02894_b200 import synth

    if name.startswith("C1"):
        return synth.synth_mask("sphere", (64, 64, 64), radius=24)
    if name.startswith("C5"):
        return synth.thin_slab()
    return synth.kits_like(tumor_mm=30.0)


@pytest.mark.parametrize("name", ["C1_sphere64_r24", "C5_thin_slab", "C2_kits_R30"])
def test_big_configs(sc, golden, name, cuda_device):
    case = next(c for c in golden["big"] if c["name"] == name)
    arr = _big(sc, name)
    assert hashlib.sha256(arr.tobytes()).hexdigest() == case["sha256"]
    got = sc.calculate_coefficients(arr, case["spacing"], device=cuda_device)
    assert_matches(got, case["features"], case["triangle_count"], case["active_cubes"], name)


def test_device_entry_and_shards(sc, golden, cuda_device):
    import torch

    from paper_2510_02894_b200 import synth

    case = next(c for c in golden["big"] if c["name"] == "C2_kits_R30")
    arr = synth.kits_like(tumor_mm=30.0)
    d = torch.from_numpy(arr).cuda()
    full = sc.calculate_coefficients_device(d, case["spacing"])
    assert_matches(full, case["features"], case["triangle_count"], case["active_cubes"], "dev")
    sq = torch.zeros(4, dtype=torch.float64, device="cuda")
    best = torch.zeros(4, dtype=torch.float64, device="cuda")
    for shard in range(3):
        part = sc.calculate_coefficients_shard(d, case["spacing"], shard, 3, sq)
        assert part.vertex_count == full.vertex_count
        torch.maximum(best, sq, out=best)
    got = [math.sqrt(v) for v in best.cpu().tolist()]
    assert got == [full.max_3d_diameter, full.max_2d_diameter_xy, full.max_2d_diameter_xz,
                   full.max_2d_diameter_yz]


def test_batch_entry(sc, golden, golden_arrays, cuda_device):
    cases = golden["cases"][:12]
    outs = sc.calculate_coefficients_batch([golden_arrays[c["mask_key"]] for c in cases],
                                           [c["spacing"] for c in cases], device=cuda_device)
    for c, got in zip(cases, outs):
        assert_matches(got, c["features"], c["triangle_count"], c["active_cubes"], c["name"])


def test_device_batch_pipeline(sc, golden, golden_arrays, cuda_device):
    import torch

    cases = golden["cases"][:10]
    ds = [torch.from_numpy(np.ascontiguousarray(golden_arrays[c["mask_key"]])).cuda()
          for c in cases]
    outs = sc.calculate_coefficients_device_batch(ds, [c["spacing"] for c in cases],
                                                  stream=torch.cuda.current_stream())
    for c, got in zip(cases, outs):
        assert_matches(got, c["features"], c["triangle_count"], c["active_cubes"], c["name"])
    # an empty ROI inside a batch fails alone
    ds2 = [ds[0], torch.zeros((4, 4, 4), dtype=torch.uint8, device="cuda"), ds[1]]
    with pytest.raises(sc.EmptyRoi):
        sc.calculate_coefficients_device_batch(ds2, [cases[0]["spacing"], (1, 1, 1),
                                                     cases[1]["spacing"]])


def test_repeat_calls_deterministic(sc, cuda_device):
    from paper_2510_02894_b200 import synth

    arr = synth.thin_slab()
    a = sc.calculate_coefficients(arr, (0.5, 0.5, 5.0))
    b = sc.calculate_coefficients(arr, (0.5, 0.5, 5.0))
    assert a.to_dict() == b.to_dict()
    assert (a.triangle_count, a.active_cubes) == (b.triangle_count, b.active_cubes)


def test_pruning_and_pass1_variants_identical(sc, golden, golden_arrays, cuda_device):
    """Work pruning, the FFMA/FFMA2 pass-1 variants, graph replay and the
    pack-fused bbox never change a result."""
    from paper_2510_02894_b200 import _native, synth

    cases = [(golden_arrays[c["mask_key"]], c["spacing"]) for c in golden["cases"]]
    cases.append((synth.thin_slab(), (0.5, 0.5, 5.0)))
    cases.append((synth.kits_like(tumor_mm=60.0), (0.8, 0.8, 1.0)))
    base = [sc.calculate_coefficients(a, sp).to_dict() for a, sp in cases]
    for opt, val in (("prune", 0), ("pass1_packed", 0), ("graphs", 0), ("fused_bbox", 0),
                     ("pack_skip", 0), ("pack_tma_single", 1),
                     ("fused_bbox_single", 1)):
        with _native.thread_options(**{opt: val}):
            for (a, sp), want in zip(cases, base):
                assert sc.calculate_coefficients(a, sp).to_dict() == want, opt
    _native.set_option("prune", 1)
    sc.calculate_coefficients(cases[-1][0], cases[-1][1])
    d = _native.last_diagnostics(cuda_device)
    assert 0 < d["work_units"] < d["total_units"]  # the KiTS-like ROI actually prunes


def test_batch_launch_options_identical(sc, golden, golden_arrays, cuda_device):
    """Launch-shape options of the batch pipeline (grid divisor, programmatic
    dependent launch, stage events, slot count, pack grid, sparse bit volume)
    never change a result, on device and host batches."""
    import torch

    from paper_2510_02894_b200 import _native, synth

    cases = [(golden_arrays[c["mask_key"]], c["spacing"]) for c in golden["cases"][:8]]
    cases.append((synth.thin_slab(), (0.5, 0.5, 5.0)))
    cases.append((synth.kits_like(tumor_mm=45.0), (0.8, 0.8, 1.0)))
    want = [sc.calculate_coefficients(a, sp).to_dict() for a, sp in cases]
    ds = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a, _ in cases]
    sps = [sp for _, sp in cases]
    for opt, val in (("grid_div", 1), ("grid_div", 2), ("pdl", 1), ("batch_stage_times", 1),
                     ("slots", 8), ("slots", 1), ("pack_mode", 3), ("sparse_bits", 0),
                     ("fork", 0), ("pack_tma", 0), ("pack_tma", 2), ("zero_copy", 0),
                     ("fused_bbox", 0), ("pack_skip", 0), ("pack_threads", 128),
                     ("pack_stages", 6), ("pack_tile", 16), ("pack_tile", 8), ("pack_prio", 0),
                     ("slots", 64), ("pack_chain", 0)):
        with _native.thread_options(**{opt: val}):
            got = sc.calculate_coefficients_device_batch(ds * 2, sps * 2)
            assert [g.to_dict() for g in got] == want * 2, (opt, val)
            got = sc.calculate_coefficients_batch([a for a, _ in cases], sps)
            assert [g.to_dict() for g in got] == want, (opt, val)


def test_graph_replay_sees_new_mask_contents(sc, cuda_device):
    """A cached CUDA graph keyed on the same device pointer must read the new
    contents of that buffer (device entry reuse, as in a serving loop)."""
    import torch

    from paper_2510_02894_b200 import synth

    a = synth.synth_mask("sphere", (64, 64, 64), radius=20)
    b = synth.synth_mask("ellipsoid", (64, 64, 64), semi_axes=(25, 15, 10))
    d = torch.from_numpy(a).cuda()
    ra = sc.calculate_coefficients_device(d, (1.0, 1.0, 1.0))
    ra2 = sc.calculate_coefficients_device(d, (1.0, 1.0, 1.0))  # graph replay
    d.copy_(torch.from_numpy(b))
    rb = sc.calculate_coefficients_device(d, (1.0, 1.0, 1.0))
    assert ra.to_dict() == ra2.to_dict()
    assert rb.to_dict() == sc.calculate_coefficients(b, (1.0, 1.0, 1.0)).to_dict()
    assert rb.to_dict() != ra.to_dict()


def _hull_max_sq(pts, oracle_mod):
    """Reference-arithmetic max squared distance over the convex-hull vertices
    of pts (n, d); the maximum pair of a point set always lies on its hull."""
    from scipy.spatial import ConvexHull, QhullError

    if len(pts) < 2:
        return 0.0
    try:
        idx = ConvexHull(pts).vertices if len(pts) > pts.shape[1] + 1 else np.arange(len(pts))
    except QhullError:  # degenerate (collinear / coplanar): use every point
        idx = np.arange(len(pts))
    sub = pts[np.sort(idx)]
    cols = [sub[:, k] for k in range(sub.shape[1])] + [np.zeros(len(sub))] * (3 - sub.shape[1])
    return oracle_mod.diameters(*cols, threads=0)[0] ** 2


@pytest.mark.timeout(900)
def test_c3_noisy_ellipsoid(sc, oracle_mod, cuda_device):
    """C3 (512^3, ~2M vertices, 1.93e12 pairs): counts, area and volume against
    the oracle's full marching cubes; diameters against the reference
    arithmetic on convex-hull subsets ("hull-subset parity")."""
    from paper_2510_02894_b200 import synth

    arr = synth.noisy_ellipsoid(512)
    assert int(arr.sum()) == 30765643
    got = sc.calculate_coefficients(arr, (1.0, 1.0, 1.0), device=cuda_device)
    assert got.vertex_count == 1963474 and got.triangle_count == 3870288
    mesh = oracle_mod.marching_cubes(arr)
    assert mesh.vertex_count == got.vertex_count and mesh.triangle_count == got.triangle_count
    assert got.active_cubes == oracle_mod.active_cubes(arr)
    assert rel_err(got.surface_area, oracle_mod.surface_area(mesh)) <= REL_TOL
    assert rel_err(got.mesh_volume, oracle_mod.mesh_volume(mesh)) <= REL_TOL
    pts = np.column_stack((mesh.xs, mesh.ys, mesh.zs))
    d3 = math.sqrt(_hull_max_sq(pts, oracle_mod))
    assert rel_err(got.max_3d_diameter, d3) <= 1e-12
    for col, key, inplane in ((2, "max_2d_diameter_xy", (0, 1)), (1, "max_2d_diameter_xz", (0, 2)),
                              (0, "max_2d_diameter_yz", (1, 2))):
        order = np.argsort(pts[:, col], kind="stable")
        vals = pts[order, col]
        cuts = np.flatnonzero(np.diff(vals)) + 1
        best = 0.0
        for grp in np.split(order, cuts):
            if len(grp) >= 2:
                best = max(best, _hull_max_sq(pts[grp][:, inplane], oracle_mod))
        assert rel_err(getattr(got, key), math.sqrt(best)) <= 1e-12, key
    # SURVEY 8e pair-grid split: the shard entry at N = 2 / 4 / 8, run in
    # sequence and MAX-combined, equals the full call bit for bit.
    import torch

    d = torch.from_numpy(arr).cuda()
    full = sc.calculate_coefficients_device(d, (1.0, 1.0, 1.0)).to_dict()
    assert full == got.to_dict()
    sq = torch.zeros(4, dtype=torch.float64, device="cuda")
    for n in (2, 4, 8):
        best = torch.zeros(4, dtype=torch.float64, device="cuda")
        for shard in range(n):
            part = sc.calculate_coefficients_shard(d, (1.0, 1.0, 1.0), shard, n, sq)
            assert part.vertex_count == full["VertexCount"]
            assert part.triangle_count == got.triangle_count
            torch.maximum(best, sq, out=best)
        comb = [math.sqrt(v) for v in best.cpu().tolist()]
        assert comb == [full[k] for k in DIAM_KEYS], n


_OVERFLOW_SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1])
from paper_2510_02894_b200 import _native, synth
import paper_2510_02894_b200 as sc
_native.set_option(sys.argv[2], int(sys.argv[3]))  # before any slot exists: far too small
arr = synth.thin_slab()
outs = sc.calculate_coefficients_batch([arr] * 3, [(0.5, 0.5, 5.0)] * 3)
one = sc.calculate_coefficients(arr, (0.5, 0.5, 5.0))
print(json.dumps([o.to_dict() | {"T": o.triangle_count, "A": o.active_cubes} for o in outs + [one]]))
"""


@pytest.mark.parametrize("option,value", [("dcap", 1000), ("wcap", 4)])
def test_capacity_overflow_rerun(golden, cuda_device, option, value):
    """More vertices (dcap) or surviving 3-D chunk pairs (wcap) than the
    buffers hold: the device reports the overflow, the host re-runs with exact
    sizes, results are unchanged (fresh process so the slots start small)."""
    import json
    import subprocess
    import sys

    from conftest import ROOT

    case = next(c for c in golden["big"] if c["name"] == "C5_thin_slab")
    out = subprocess.run([sys.executable, "-c", _OVERFLOW_SCRIPT, ROOT, option, str(value)],
                         capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    for rec in json.loads(out.stdout.strip().splitlines()[-1]):
        assert rec["VertexCount"] == case["features"]["VertexCount"]
        assert rec["T"] == case["triangle_count"] and rec["A"] == case["active_cubes"]
        for k in DIAM_KEYS:
            assert rec[k] == case["features"][k], k


def test_canonical_mesh_bit_exact(sc, golden, golden_arrays, cuda_device):
    """marching_cubes on the GPU == the reference's TriangleMesh, element by
    element: vertex order (first reference), coordinates, triangles; and the
    mesh measures == the reference's surface_area / mesh_volume bit for bit."""
    n = 0
    for case in golden["cases"]:
        if "verts_key" not in case:
            continue
        vol = sc.MaskVolume.from_array(golden_arrays[case["mask_key"]], case["spacing"])
        mesh = sc.marching_cubes(vol)
        want = golden_arrays[case["verts_key"]]
        got = np.column_stack((mesh.xs, mesh.ys, mesh.zs))
        assert np.array_equal(got, want), case["name"]
        assert mesh.triangle_count == case["triangle_count"]
        n += 1
    assert n >= 10


def test_canonical_mesh_against_oracle(sc, oracle_mod, cuda_device):
    from paper_2510_02894_b200 import synth

    for arr, sp in ((synth.synth_mask("sphere", (64, 64, 64), radius=24), (1.0, 1.0, 1.0)),
                    (synth.thin_slab(), (0.5, 0.5, 5.0)),
                    (synth.kits_like(tumor_mm=30.0), (0.8, 0.8, 1.0))):
        mesh = sc.marching_cubes(sc.MaskVolume.from_array(arr, sp))
        ref = oracle_mod.marching_cubes(arr, sp)
        assert np.array_equal(mesh.xs, ref.xs) and np.array_equal(mesh.ys, ref.ys)
        assert np.array_equal(mesh.zs, ref.zs)
        assert np.array_equal(mesh.triangles, ref.triangles)
        assert sc.surface_area(mesh) == oracle_mod.surface_area(ref)
        assert sc.mesh_volume(mesh) == oracle_mod.mesh_volume(ref)


def test_mesh_measure_small_meshes(sc, cuda_device):
    # pkg/tests/test_features.py:47-59
    m = sc.TriangleMesh(xs=np.array([0.0, 1.0, 0.0]), ys=np.array([0.0, 0.0, 1.0]),
                        zs=np.zeros(3), triangles=np.array([[0, 1, 2]], np.int32))
    assert sc.surface_area(m) == pytest.approx(0.5, abs=1e-15)
    e = sc.TriangleMesh(xs=np.zeros(0), ys=np.zeros(0), zs=np.zeros(0),
                        triangles=np.zeros((0, 3), np.int32))
    assert sc.surface_area(e) == 0.0 and sc.mesh_volume(e) == 0.0


def test_mesh_dump_formats(sc, tmp_path, cuda_device):
    vol = sc.MaskVolume.from_array(sc.synth_mask("box", (3, 3, 3), lo=(1, 1, 1), hi=(1, 1, 1)))
    mesh = sc.marching_cubes(vol)
    sc.mesh_dump(mesh, tmp_path / "m.off")
    lines = (tmp_path / "m.off").read_text().splitlines()
    assert lines[0] == "OFF" and lines[1] == "6 8 0" and len(lines) == 2 + 6 + 8
    sc.mesh_dump(mesh, tmp_path / "m.stl")
    assert (tmp_path / "m.stl").stat().st_size == 84 + 50 * 8


def _offset_blobs(seed):
    """Small occupied regions far from the grid origin (large slab offsets) at
    spacings whose fp64 coordinates round differently at different offsets."""
    rng = np.random.default_rng(seed)
    nz, ny, nx = 70, 90, 64 + 8 * seed
    arr = np.zeros((nz, ny, nx), dtype=np.uint8)
    for _ in range(3):
        c = rng.uniform([40, 55, 10], [nz - 6, ny - 6, nx - 10])
        r = rng.uniform(2, 5, 3)
        z, y, x = np.ogrid[:nz, :ny, :nx]
        arr |= (((z - c[0]) / r[0]) ** 2 + ((y - c[1]) / r[1]) ** 2
                + ((x - c[2]) / r[2]) ** 2 <= 1).astype(np.uint8)
    arr[nz - 1, ny - 1, nx - 1] = 1  # touches the far grid corner
    return arr


def test_host_crop_is_exact(sc, oracle_mod, cuda_device):
    """Host entries copy only the occupied z/y slab and add its origin back on
    the device: results identical to the uncropped copy, to the device-resident
    entry and to the oracle (diameters bit-exact at odd spacings)."""
    import torch

    from paper_2510_02894_b200 import _native

    cases = [(_offset_blobs(s), sp) for s, sp in
             ((0, (0.7, 0.3, 1.3)), (1, (0.1, 0.9, 3.7)), (2, (1.1, 1.1, 0.45)))]
    cases.append((np.pad(np.ones((1, 1, 1), np.uint8), ((37, 2), (5, 60), (3, 9))),
                  (0.37, 0.61, 2.9)))
    try:
        for arr, sp in cases:
            z0, z1, y0, y1 = _native.occupied_slab(arr)
            # host pack: the slab's bits cross PCIe into the bit volume
            _native.set_option("host_pack", 1)
            _native.set_option("host_split", 0)
            packed = sc.calculate_coefficients(arr, sp, device=cuda_device)
            assert packed.h2d_bytes == 4 * ((arr.shape[2] + 31) // 32) * (z1 - z0 + 1) * (y1 - y0 + 1)
            _native.set_option("host_pack", 0)
            _native.set_option("host_split", 0)
            cropped = sc.calculate_coefficients(arr, sp, device=cuda_device)
            assert cropped.h2d_bytes == (z1 - z0 + 1) * (y1 - y0 + 1) * arr.shape[2]
            assert packed.to_dict() == cropped.to_dict()
            assert (packed.triangle_count, packed.active_cubes) == \
                   (cropped.triangle_count, cropped.active_cubes)
            # split read: leading slices cross PCIe unscanned, the rest is cropped
            for pct in (30, 60, 90):
                _native.set_option("host_split", pct)
                split = sc.calculate_coefficients(arr, sp, device=cuda_device)
                assert split.to_dict() == cropped.to_dict(), pct
                assert (split.triangle_count, split.active_cubes) == \
                       (cropped.triangle_count, cropped.active_cubes)
            _native.set_option("host_split", -1)
            _native.set_option("host_pack", -1)
            dev = sc.calculate_coefficients_device(torch.from_numpy(arr).cuda(), sp)
            _native.set_option("host_crop", 0)
            full = sc.calculate_coefficients(arr, sp, device=cuda_device)
            _native.set_option("host_crop", 1)
            assert full.h2d_bytes == arr.size
            assert cropped.to_dict() == full.to_dict() == dev.to_dict()
            assert (cropped.triangle_count, cropped.active_cubes) == \
                   (full.triangle_count, full.active_cubes)
            want = oracle_mod.extract_features(arr, sp)
            rec = cropped.to_dict()
            for k in DIAM_KEYS:
                assert rec[k] == want[k], (k, rec[k], want[k])
            assert cropped.triangle_count == want["triangle_count"]
            for k in ("MeshVolume", "SurfaceArea"):
                assert rel_err(rec[k], want[k]) <= 1e-12
        # an all-background mask is an EmptyRoi whichever part the host scanned
        for pack, pct in ((1, 0), (-1, -1), (0, 0), (0, 50)):
            _native.set_option("host_pack", pack)
            _native.set_option("host_split", pct)
            with pytest.raises(sc.EmptyRoi):
                sc.calculate_coefficients(np.zeros((40, 30, 64), np.uint8), (1, 1, 1))
        # the pipelined host batch packs / crops / splits too
        for pack, pct in ((1, 0), (-1, -1), (0, -1), (0, 50)):
            _native.set_option("host_pack", pack)
            _native.set_option("host_split", pct)
            outs = sc.calculate_coefficients_batch([a for a, _ in cases] * 3,
                                                   [s for _, s in cases] * 3, device=cuda_device)
            for (arr, sp), o in zip(cases * 3, outs):
                assert o.to_dict() == sc.calculate_coefficients(arr, sp).to_dict()
    finally:
        _native.set_option("host_crop", 1)
        _native.set_option("host_split", -1)
        _native.set_option("host_pack", -1)


def _blob_mask(seed):
    """Seeded multi-blob masks of varied shape (round, elongated, flat, tiny)
    with vertex counts that are not multiples of the 64 / 128 chunk sizes."""
    from paper_2510_02894_b200 import synth

    rng = np.random.default_rng(seed)
    dims = tuple(int(v) for v in rng.integers(24, 90, 3))  # (nx, ny, nz)
    arr = np.zeros(dims[::-1], dtype=np.uint8)
    for _ in range(int(rng.integers(1, 7))):
        semi = rng.uniform(0.6, 0.45 * min(dims), 3) * rng.choice([1.0, 0.25], 3, p=[0.7, 0.3])
        c = [rng.uniform(semi[a] * 0 + 1, dims[a] - 2) for a in range(3)]
        synth.ellipsoid_into(arr, c, np.maximum(semi, 0.6))
    if not arr.any():
        arr[dims[2] // 2, dims[1] // 2, dims[0] // 2] = 1
    sp = tuple(float(v) for v in rng.choice([0.5, 0.7, 0.8, 1.0, 1.3, 2.5, 5.0], 3))
    return arr, sp


def test_sub_pair_pruning_random_masks(sc, oracle_mod, cuda_device):
    """Exact pruning with 64 x 64 sub-pair masks: 24 seeded multi-blob masks,
    pruned == unpruned == oracle (diameters bit-exact, counts exact)."""
    from paper_2510_02894_b200 import _native

    try:
        for seed in range(24):
            arr, sp = _blob_mask(seed)
            _native.set_option("prune", 1)
            got = sc.calculate_coefficients(arr, sp, device=cuda_device)
            _native.set_option("prune", 0)
            full = sc.calculate_coefficients(arr, sp, device=cuda_device)
            assert got.to_dict() == full.to_dict(), seed
            want = oracle_mod.extract_features(arr, sp, threads=0)
            rec = got.to_dict()
            assert rec["VertexCount"] == want["VertexCount"], seed
            assert got.triangle_count == want["triangle_count"], seed
            for k in DIAM_KEYS:
                assert rec[k] == want[k], (seed, k, rec[k], want[k])
            # the device volume is the exact K sx sy sz / 48; the reference's
            # fp64 triangle sums drift by ~1e-12 relative on small meshes
            for k in ("MeshVolume", "SurfaceArea"):
                assert rel_err(rec[k], want[k]) <= REL_TOL, (seed, k)
    finally:
        _native.set_option("prune", 1)


@pytest.mark.timeout(600)
def test_randomized_stress_parity(cuda_device):
    """tools/stress_parity.py: 60 seeded masks of varied kind (random voxels,
    blobs, sheets, face-touching boxes, nonbinary singles), size, alignment and
    spacing through the host single call, the host batch (crop / split) and the
    device batch, against the oracle."""
    import subprocess
    import sys

    from conftest import ROOT

    r = subprocess.run([sys.executable, "tools/stress_parity.py", "60", "11"], cwd=ROOT,
                       capture_output=True, text=True, timeout=580)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "stress parity ok" in r.stdout


def test_stage_times_from_device_timestamps(sc, cuda_device):
    """mesh_ms / diameters_ms without event nodes (device %globaltimer stamps)
    are positive and consistent with the event-timed values; all event levels
    give identical results."""
    from paper_2510_02894_b200 import _native, synth

    arr = synth.kits_like(128, 128, 96, (0.8, 0.8, 1.0), 20.0)
    recs = {}
    try:
        for lvl in (0, 1, 2):
            _native.set_option("stage_times", lvl)
            c = sc.calculate_coefficients(arr, (0.8, 0.8, 1.0))
            c = sc.calculate_coefficients(arr, (0.8, 0.8, 1.0))
            assert c.mesh_ms > 0 and c.diameters_ms > 0, lvl
            assert c.total_ms >= c.mesh_ms + c.diameters_ms
            recs[lvl] = c.to_dict()
            times = _native.last_kernel_times(cuda_device)
            assert (times["pack_ms"] > 0) == (lvl == 2)
    finally:
        _native.set_option("stage_times", 0)
    assert recs[0] == recs[1] == recs[2]
    outs = sc.calculate_coefficients_batch([arr] * 4, [(0.8, 0.8, 1.0)] * 4)
    assert all(o.mesh_ms > 0 and o.diameters_ms > 0 for o in outs)


def test_two_level_filter_list_sized_for_every_super_pair(sc, cuda_device):
    """with a small diameter-side capacity (option dcap) the ROI
    is re-run with exact sizes; its super-pair list must still hold every
    super pair the two-level filter can list (pruning off lists them all),
    or the maximum pair could be skipped silently."""
    from paper_2510_02894_b200 import _native, synth

    a = synth.kits_like(512, 512, 300, (0.8, 0.8, 1.0), 45.0)  # C(C+1)/2 in (2^16, 2^22]
    want = sc.calculate_coefficients(a, (0.8, 0.8, 1.0)).to_dict()
    for opts in ({"dcap": 256, "prune": 0}, {"dcap": 256}, {"dcap": 4096, "prune": 0}):
        with _native.thread_options(**opts):
            got = sc.calculate_coefficients(a, (0.8, 0.8, 1.0)).to_dict()
        assert got == want, opts


def test_cloud_diameters_grid_covers_every_tile_pair(sc, cuda_device):
    """sc_diameters walks the T(T+1)/2 tile pairs with a bounded,
    grid-stride launch (SMs x 8 blocks); a cloud of 2^20 points (4096 tiles,
    8.4e6 tile pairs, ~7 K per block) whose extreme pair sits in the last
    tile must still be found."""
    rng = np.random.default_rng(5)
    n = 1 << 20
    xs = rng.uniform(0, 10, n)
    ys = rng.uniform(0, 10, n)
    zs = rng.uniform(0, 10, n)
    xs[-1], ys[-1], zs[-1] = 100.0, 100.0, 100.0  # far point in the last tile
    xs[-2], ys[-2], zs[-2] = -100.0, -100.0, 100.0  # same z: also the XY maximum
    got = sc.diameters(xs, ys, zs)
    d3 = math.sqrt(200.0 ** 2 + 200.0 ** 2)
    assert got[0] == d3 and got[1] == d3


def _lesion_field(seed, sp, diagonal):
    """Many small lesions (radius 1.2-3 voxels) spread over a 512 x 512 field:
    each plane family's maximum is a lesion diameter (a few mm) while the
    pass-1 frame spans the whole field (R ~ 190 mm), the case where a margin
    relative to the family maximum would not cover the fp32 error."""
    rng = np.random.default_rng(seed)
    nz = 14
    arr = np.zeros((nz, 512, 512), dtype=np.uint8)
    n = 48
    if diagonal:  # no two lesions share an x or y row: XZ / YZ maxima = one lesion
        t = np.sort(rng.choice(np.arange(10, 500, 9), size=n, replace=False))
        cx, cy = t.astype(float), t[::-1].astype(float) if seed % 2 else t.astype(float)
    else:
        cx, cy = rng.uniform(10, 500, n), rng.uniform(10, 500, n)
    zz, yy, xx = np.ogrid[:nz, :16, :16]
    for x, y in zip(cx, cy):
        r = rng.uniform(1.2, 3.0)
        z = rng.uniform(4, nz - 5)
        x0, y0 = int(x) - 8, int(y) - 8
        blob = ((zz - z) ** 2 + (yy - (y - y0)) ** 2 + (xx - (x - x0)) ** 2) <= r * r
        arr[:, y0:y0 + 16, x0:x0 + 16] |= blob.astype(np.uint8)
    return arr, sp


def test_planar_recheck_margin_on_spread_lesions(sc, oracle_mod, cuda_device):
    """adversarial multi-lesion masks at 0.7421875 and 0.8
    mm in-plane spacing (random and row-disjoint diagonal placements): the
    re-check threshold is absolute in the frame extent (refine_tau), so every
    diameter -- the XZ / YZ families above all -- is the reference's bit for
    bit, through the single call and the device batch."""
    import torch

    cases = []
    for seed in range(8):
        for sp in ((0.7421875, 0.7421875, 1.0), (0.8, 0.8, 1.0)):
            cases.append(_lesion_field(seed, sp, diagonal=seed >= 4))
    wants = [oracle_mod.extract_features(a, sp, threads=0) for a, sp in cases]
    ds = [torch.from_numpy(a).cuda() for a, _ in cases]
    batch = sc.calculate_coefficients_device_batch(ds, [sp for _, sp in cases])
    for (a, sp), want, b in zip(cases, wants, batch):
        got = sc.calculate_coefficients(a, sp).to_dict()
        assert got == b.to_dict()
        assert got["VertexCount"] == want["VertexCount"]
        for k in DIAM_KEYS:
            assert got[k] == want[k], (k, sp, got[k], want[k])


def test_c4_sample_against_reference_goldens(sc, cuda_device):
    """12 of C4's 300 varied KiTS-like masks (every 25th of
    kits_batch_params(300, 2025): nz 230-597, in-plane spacing 0.6-0.9 mm,
    V 56 K - 184 K) through the device batch entry (mixed dims in one call)
    and the host batch entry, against the records the reference itself
    produced (tools/make_golden_c4.py): counts exact, diameters bit-exact,
    area / volume within the north_star tolerance (1e-6 relative)."""
    import hashlib
    import json
    import os

    import torch

    from conftest import GOLD
    from paper_2510_02894_b200 import synth

    with open(os.path.join(GOLD, "c4_golden.json")) as fh:
        gold = json.load(fh)["cases"]
    params = synth.kits_batch_params(300, 2025)
    masks, sps = [], []
    for g in gold:
        m = synth.kits_from_params(params[g["index"]])
        assert hashlib.sha256(m.tobytes()).hexdigest() == g["sha256"], g["index"]
        masks.append(m)
        sps.append(tuple(g["spacing"]))
    ds = [torch.from_numpy(m).cuda() for m in masks]
    dev = sc.calculate_coefficients_device_batch(ds, sps)
    del ds
    host = sc.calculate_coefficients_batch(masks, sps)
    for g, d, h in zip(gold, dev, host):
        want = g["features"]
        for got in (d, h):
            rec = got.to_dict()
            assert rec["VertexCount"] == want["VertexCount"], g["index"]
            assert got.triangle_count == g["triangle_count"], g["index"]
            assert got.active_cubes == g["active_cubes"], g["index"]
            for k in DIAM_KEYS:
                assert rec[k] == want[k], (g["index"], k, rec[k], want[k])
            for k in ("MeshVolume", "SurfaceArea"):
                assert rel_err(rec[k], want[k]) <= REL_TOL, (g["index"], k)


def test_large_face_grid_against_oracle(sc, oracle_mod, cuda_device):
    """no up-front refusal of large grid faces (2048 x 2048
    slices); the planar chunk-index width is checked per plane at run time.
    A 2048 x 2048 x 8 mask with blobs spread over the slice equals the oracle
    (counts exact, diameters bit-exact)."""
    rng = np.random.default_rng(3)
    arr = np.zeros((8, 2048, 2048), np.uint8)
    zz, yy, xx = np.ogrid[:8, :24, :24]
    for _ in range(40):
        y0, x0 = (int(v) for v in rng.integers(8, 2048 - 32, size=2))
        r = rng.uniform(2.0, 3.4)
        blob = ((zz - 3.5) ** 2 + (yy - 12) ** 2 + (xx - 12) ** 2) <= r * r
        arr[:, y0:y0 + 24, x0:x0 + 24] |= blob.astype(np.uint8)
    sp = (0.3, 0.3, 2.0)
    want = oracle_mod.extract_features(arr, sp, threads=0)
    for got in (sc.calculate_coefficients(arr, sp),
                sc.calculate_coefficients_batch([arr, arr], [sp, sp])[1]):
        rec = got.to_dict()
        assert rec["VertexCount"] == want["VertexCount"]
        assert got.triangle_count == want["triangle_count"]
        for k in DIAM_KEYS:
            assert rec[k] == want[k], k
        for k in ("MeshVolume", "SurfaceArea"):
            assert rel_err(rec[k], want[k]) <= REL_TOL, k


def _tie_masks():
    """Shapes whose maximum pair is massively tied or sits exactly at the
    extremes-based lower bound, at odd spacings: solid boxes (four tied space
    diagonals and many tied in-plane diagonals), a thin plate, two isolated
    voxels far apart, an L, a hollow shell and a one-voxel-thick ring."""
    out = []
    a = np.zeros((24, 24, 24), np.uint8); a[2:22, 2:22, 2:22] = 1
    out.append(("cube", a, (1.0, 1.0, 1.0)))
    a = np.zeros((17, 11, 34), np.uint8); a[2:15, 2:9, 3:31] = 1
    out.append(("box", a, (0.7, 1.3, 2.1)))
    a = np.zeros((5, 60, 60), np.uint8); a[2, 3:57, 3:57] = 1
    out.append(("plate", a, (0.8, 0.8, 5.0)))
    a = np.zeros((40, 40, 64), np.uint8); a[3, 4, 5] = 1; a[36, 35, 58] = 1
    out.append(("two_voxels", a, (0.9, 0.6, 1.1)))
    a = np.zeros((30, 30, 30), np.uint8); a[2:28, 2:6, 2:28] = 1; a[2:6, 2:28, 2:28] = 1
    out.append(("l_shape", a, (1.0, 0.5, 2.0)))
    zz, yy, xx = np.mgrid[:48, :48, :48]
    r = np.sqrt((zz - 23.5) ** 2 + (yy - 23.5) ** 2 + (xx - 23.5) ** 2)
    out.append(("shell", ((r > 17) & (r < 20)).astype(np.uint8), (0.75, 0.75, 1.5)))
    yy, xx = np.mgrid[:64, :64]
    ring = (np.abs(np.hypot(yy - 31.5, xx - 31.5) - 25) < 0.75).astype(np.uint8)
    a = np.zeros((3, 64, 64), np.uint8); a[1] = ring
    out.append(("ring", a, (0.8, 0.8, 3.0)))
    return out


def test_reach_filter_on_tied_maxima(sc, oracle_mod, cuda_device):
    """Pass 1's vertex reach filter (and the box pruning) on shapes whose
    maximum is tied many times or equals the extremes' lower bound: pruned
    (filter on) == unpruned (filter off) == oracle, bit for bit."""
    from paper_2510_02894_b200 import _native

    try:
        for name, arr, sp in _tie_masks():
            _native.set_option("prune", 1)
            got = sc.calculate_coefficients(arr, sp, device=cuda_device)
            _native.set_option("prune", 0)
            full = sc.calculate_coefficients(arr, sp, device=cuda_device)
            assert got.to_dict() == full.to_dict(), name
            want = oracle_mod.extract_features(arr, sp, threads=0)
            assert_matches(got, want, want["triangle_count"], want["active_cubes"], name)
    finally:
        _native.set_option("prune", 1)
