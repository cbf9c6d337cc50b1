"""Golden records for a sample of the C4 batch, by running
the REFERENCE (numba, /root/reference/pkg via a writable copy).

For every 25th mask of synth.kits_batch_params(300, 2025) (12 masks of mixed
nz and spacing) it stores the mask's sha256, the reference's 7-key record
(extract_features with the "parallel" backend, features.py:224-265), the
reference's triangle count (marching_cubes(vol).triangle_count, mesh.py:50-52)
and the active-cube count restated from _cell_case (mesh.py:103-128) ->
tests/golden/c4_golden.json.  tests/test_gpu_parity.py regenerates the masks
(deterministic, the hash is checked first) and runs them through the device
batch entry.

usage: python tools/make_golden_c4.py
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from make_golden import active_cubes, ref_module  # noqa: E402

from paper_2510_02894_b200 import synth  # noqa: E402


def main():
    ref = ref_module()
    params = synth.kits_batch_params(300, 2025)
    out = {"source": "reference shapecore.extract_features(parallel) + marching_cubes, "
                     "tools/make_golden_c4.py", "params": "kits_batch_params(300, 2025)",
           "cases": []}
    for i in range(0, 300, 25):
        p = params[i]
        m = synth.kits_from_params(p)
        nz, ny, nx = m.shape
        vol = ref.MaskVolume(dims=(nx, ny, nz), spacing=tuple(p["sp"]), data=m.reshape(-1))
        t0 = time.time()
        feats, _ = ref.extract_features(vol, ref.resolve_backend("parallel"))
        tri = ref.marching_cubes(vol).triangle_count
        rec = feats.to_dict() if hasattr(feats, "to_dict") else dict(feats.as_dict())
        out["cases"].append({"index": i, "dims": [nx, ny, nz], "spacing": list(p["sp"]),
                             "sha256": hashlib.sha256(m.tobytes()).hexdigest(),
                             "features": rec, "triangle_count": int(tri),
                             "active_cubes": active_cubes(m)})
        print(i, (nx, ny, nz), rec["VertexCount"], f"{time.time() - t0:.1f}s", flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "c4_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
