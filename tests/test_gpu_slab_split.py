"""GPU parity of the two-phase (slab-split) shard entry, SURVEY.md 8e.

sc_shard_mesh runs marching cubes over one shard's share of the cell layers;
the int64 partials are summed and the vertex keys concatenated (what the NCCL
all-reduce / all-gather do across GPUs), then sc_shard_diameters evaluates one
shard of the pair grid.  All shards run one after another on this GPU
(sharding.simulate_slab_shards) and the combined record must equal the
single call bit for bit -- counts, area, volume and all four diameters -- and
the reference goldens.
"""

import numpy as np
import pytest

from conftest import REL_TOL, rel_err

pytestmark = pytest.mark.gpu

KEYS = ("VertexCount", "MeshVolume", "SurfaceArea", "Maximum3DDiameter",
        "Maximum2DDiameterXY", "Maximum2DDiameterXZ", "Maximum2DDiameterYZ")


def _full(sc, d, sp):
    c = sc.calculate_coefficients_device(d, sp)
    return c.to_dict() | {"triangle_count": c.triangle_count, "active_cubes": c.active_cubes}


def _check_equal(got, full, label):
    for k in KEYS + ("triangle_count", "active_cubes"):
        assert got[k] == full[k], (label, k, got[k], full[k])


def test_golden_cases_all_shard_counts(sc, golden, golden_arrays, cuda_device):
    import torch

    from paper_2510_02894_b200 import sharding

    for case in golden["cases"][:24]:
        arr = np.ascontiguousarray(golden_arrays[case["mask_key"]], dtype=np.uint8)
        d = torch.from_numpy(arr).cuda()
        full = _full(sc, d, case["spacing"])
        want = case["features"]
        for n in (1, 2, 3, 5):
            got = sharding.simulate_slab_shards(d, case["spacing"], n)
            _check_equal(got, full, (case["name"], n))
            assert got["triangle_count"] == case["triangle_count"]
            assert got["active_cubes"] == case["active_cubes"]
            for k in ("Maximum3DDiameter", "Maximum2DDiameterXY", "Maximum2DDiameterXZ",
                      "Maximum2DDiameterYZ", "VertexCount"):
                assert got[k] == want[k], (case["name"], n, k)
            for k in ("MeshVolume", "SurfaceArea"):
                assert rel_err(got[k], want[k]) <= REL_TOL


def test_c3_slab_split(sc, cuda_device):
    """C3 (512^3 noisy ellipsoid, ~2M vertices) at N = 2 / 4 / 8."""
    import torch

    from paper_2510_02894_b200 import sharding, synth

    arr = synth.noisy_ellipsoid(512)
    d = torch.from_numpy(arr).cuda()
    full = _full(sc, d, (1.0, 1.0, 1.0))
    assert full["VertexCount"] == 1963474 and full["triangle_count"] == 3870288
    for n in (2, 4, 8):
        _check_equal(sharding.simulate_slab_shards(d, (1.0, 1.0, 1.0), n), full, n)


def test_kits_and_thin_slabs(sc, cuda_device):
    """C2 (KiTS-like, anisotropic spacing) and C5 (thin slabs, 0.5 x 0.5 x 5 mm)."""
    import torch

    from paper_2510_02894_b200 import sharding, synth

    cases = [(synth.kits_like(tumor_mm=30.0), (0.8, 0.8, 1.0)),
             (synth.thin_slab(), (0.5, 0.5, 5.0))]
    for arr, sp in cases:
        d = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
        full = _full(sc, d, sp)
        for n in (3, 7):
            _check_equal(sharding.simulate_slab_shards(d, sp, n), full, (arr.shape, n))


def test_more_shards_than_layers_and_errors(sc, cuda_device):
    import torch

    from paper_2510_02894_b200 import errors, sharding

    arr = np.zeros((3, 4, 32), np.uint8)
    arr[1, 2, 5] = 1
    d = torch.from_numpy(arr).cuda()
    full = _full(sc, d, (1.0, 1.0, 1.0))
    got = sharding.simulate_slab_shards(d, (1.0, 1.0, 1.0), 8)  # 4 cell layers, 8 shards
    _check_equal(got, full, "tiny")
    empty = torch.zeros((4, 4, 32), dtype=torch.uint8, device="cuda")
    with pytest.raises(errors.EmptyRoi):
        sharding.simulate_slab_shards(empty, (1.0, 1.0, 1.0), 2)
    # a wrong gathered key count is refused, not silently used
    n_sums, key_cap = sc.shard_exchange_sizes(arr.shape)
    sums = torch.empty(n_sums, dtype=torch.int64, device="cuda")
    keys = torch.empty(4 * key_cap, dtype=torch.int32, device="cuda")
    n, bbox = sc.shard_mesh(d, (1.0, 1.0, 1.0), 0, 1, sums, keys)
    assert n == full["VertexCount"] and bbox == (5, 2, 1, 5, 2, 1)
    sq4 = torch.zeros(4, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        sc.shard_diameters(sums, keys, n - 1, arr.shape, bbox, (1.0, 1.0, 1.0), 0, 1, sq4)
    # the slot is a plain ROI again afterwards
    assert _full(sc, d, (1.0, 1.0, 1.0)) == full


def test_slab_sharded_coefficients_single_rank(sc, golden, cuda_device):
    """The torch.distributed driver itself at world size 1 (no process group):
    phase 1, the (trivial) exchange, phase 2, and the MAX combine."""
    import torch

    from paper_2510_02894_b200 import sharding, synth

    case = next(c for c in golden["big"] if c["name"] == "C2_kits_R30")
    d = torch.from_numpy(synth.kits_like(tumor_mm=30.0)).cuda()
    full = _full(sc, d, case["spacing"])
    rec = sharding.slab_sharded_coefficients(d, case["spacing"])
    _check_equal(rec, full, "world 1")
    for k in ("Maximum3DDiameter", "Maximum2DDiameterXY", "Maximum2DDiameterXZ",
              "Maximum2DDiameterYZ", "VertexCount"):
        assert rec[k] == case["features"][k], k
