"""The CPU oracle (oracle/shape_oracle.c) against the reference's golden vectors.

Pins the restatement before it is trusted as the GPU checker: every small case
in tests/golden was produced by the reference (tools/make_golden.py).  Counts
and diameters must be bit-exact; area/volume are bit-exact in practice and
held to 1e-12 here (numpy's einsum may reorder a 3-term dot product).
"""

import hashlib
import math

import numpy as np
import pytest

from conftest import rel_err
from paper_2510_02894_b200 import synth

KEYS = ("MeshVolume", "SurfaceArea", "Maximum3DDiameter", "Maximum2DDiameterXY",
        "Maximum2DDiameterXZ", "Maximum2DDiameterYZ", "VertexCount")


def check_record(got, want):
    assert got["VertexCount"] == want["features"]["VertexCount"]
    assert got["triangle_count"] == want["triangle_count"]
    assert got["active_cubes"] == want["active_cubes"]
    for k in KEYS[2:6]:
        assert got[k] == want["features"][k], k
    for k in KEYS[:2]:
        assert rel_err(got[k], want["features"][k]) <= 1e-12, k


def test_small_cases_match_reference(golden, golden_arrays, oracle_mod):
    for case in golden["cases"]:
        arr = golden_arrays[case["mask_key"]]
        threads = 1 if arr.size <= 20 ** 3 else 0  # big noise masks: strip-parallel
        got = oracle_mod.extract_features(arr, case["spacing"], threads=threads)
        check_record(got, case)


def test_parallel_diameters_equal_sequential(golden, golden_arrays, oracle_mod):
    for case in golden["cases"][:20]:
        arr = golden_arrays[case["mask_key"]]
        seq = oracle_mod.extract_features(arr, case["spacing"], threads=1)
        par = oracle_mod.extract_features(arr, case["spacing"], threads=4)
        for k in KEYS:
            assert seq[k] == par[k]


def test_vertex_sets_and_order_match_reference(golden, golden_arrays, oracle_mod):
    n = 0
    for case in golden["cases"]:
        if "verts_key" not in case:
            continue
        want = golden_arrays[case["verts_key"]]
        mesh = oracle_mod.marching_cubes(golden_arrays[case["mask_key"]], case["spacing"])
        got = np.column_stack((mesh.xs, mesh.ys, mesh.zs))
        assert np.array_equal(got, want)  # canonical first-reference order too
        n += 1
    assert n >= 10


def test_known_answers(oracle_mod):
    # pkg/tests/test_features.py:62-66, 80-89; test_mesh.py:45-71
    vox = synth.synth_mask("box", (3, 3, 3), lo=(1, 1, 1), hi=(1, 1, 1))
    r = oracle_mod.extract_features(vox)
    assert r["VertexCount"] == 6 and r["triangle_count"] == 8
    assert abs(r["MeshVolume"] - 1 / 6) <= 1e-9 and abs(r["SurfaceArea"] - math.sqrt(3)) <= 1e-9
    assert (r["Maximum3DDiameter"], r["Maximum2DDiameterXY"]) == (1.0, 1.0)
    blk = synth.synth_mask("box", (4, 4, 4), lo=(1, 1, 1), hi=(2, 2, 2))
    r = oracle_mod.extract_features(blk)
    assert r["VertexCount"] == 24 and r["triangle_count"] == 44
    assert oracle_mod.diameters([0.0, 3.0], [0.0, 4.0], [0.0, 0.0]) == (5.0, 5.0, 0.0, 0.0)
    assert oracle_mod.diameters([2.5], [2.5], [2.5]) == (0.0, 0.0, 0.0, 0.0)
    with pytest.raises(ValueError):
        oracle_mod.extract_features(np.zeros((4, 4, 4), np.uint8))


def test_clouds_match_reference(golden, golden_clouds, oracle_mod):
    for c in golden["clouds"]:
        xs, ys, zs = golden_clouds[c["key"]]
        assert list(oracle_mod.diameters(xs, ys, zs)) == c["diameters"]
        assert list(oracle_mod.diameters(xs, ys, zs, threads=3)) == c["diameters"]


def test_pairwise_sum_matches_reference_fold(oracle_mod):
    rng = np.random.default_rng(5)
    for n in (0, 1, 2, 3, 7, 8, 1000, 1025):
        v = rng.normal(size=n)
        size = 1 << max(n - 1, 0).bit_length() if n else 0
        if n == 0:
            want = 0.0
        else:
            buf = np.zeros(size)
            buf[:n] = v
            while size > 1:
                size //= 2
                buf = buf[:size] + buf[size:2 * size]
            want = float(buf[0])
        assert oracle_mod.pairwise_sum(v) == want


@pytest.mark.parametrize("name", ["C1_sphere64_r24", "C5_thin_slab"])
def test_big_configs_match_reference(golden, oracle_mod, name):
    case = next(c for c in golden["big"] if c["name"] == name)
    arr = (synth.synth_mask("sphere", (64, 64, 64), radius=24) if name.startswith("C1")
           else synth.thin_slab())
    assert hashlib.sha256(arr.tobytes()).hexdigest() == case["sha256"]
    got = oracle_mod.extract_features(arr, case["spacing"], threads=0)
    check_record(got, case)


def test_oracle_matches_c4_reference_golden(oracle_mod, golden):
    """The C4 golden file (made by the reference itself) is pinned to the
    oracle too: its smallest case (V = 56,188) bit for bit on counts and
    diameters."""
    import hashlib
    import json
    import os

    from conftest import GOLD
    from paper_2510_02894_b200 import synth

    with open(os.path.join(GOLD, "c4_golden.json")) as fh:
        cases = json.load(fh)["cases"]
    g = min(cases, key=lambda c: c["features"]["VertexCount"])
    m = synth.kits_from_params(synth.kits_batch_params(300, 2025)[g["index"]])
    assert hashlib.sha256(m.tobytes()).hexdigest() == g["sha256"]
    r = oracle_mod.extract_features(m, tuple(g["spacing"]), threads=0)
    want = g["features"]
    assert r["VertexCount"] == want["VertexCount"]
    assert r["triangle_count"] == g["triangle_count"]
    assert r["active_cubes"] == g["active_cubes"]
    for k in ("Maximum3DDiameter", "Maximum2DDiameterXY", "Maximum2DDiameterXZ",
              "Maximum2DDiameterYZ"):
        assert r[k] == want[k], k
    for k in ("MeshVolume", "SurfaceArea"):
        assert abs(r[k] - want[k]) <= 1e-12 * abs(want[k]), k
