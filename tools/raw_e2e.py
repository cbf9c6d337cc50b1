"""End-to-end host-payload throughput: the C2 mask as uint8 through the host
batch entry vs the same mask stored as a typed NPY payload (int16, C and
Fortran order; float32) through the raw batch entry (host slab scan of the
typed payload, chunked pinned staging, device binarize).  VERDICT r01 #4's
bar: int16 within 1.3x of the uint8 host path.
usage: raw_e2e.py [K]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_02894_b200 as sc  # noqa: E402
from paper_2510_02894_b200 import synth  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 32
sp = (0.8, 0.8, 1.0)
m = synth.kits_like(512, 512, 600, sp, 30.0)
want = sc.calculate_coefficients(m, sp).to_dict()
res = {}


def rate(fn, n=K, reps=3):
    fn(8)
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn(n)
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) / n)
    return 1.0 / best


u8 = [m.copy() for _ in range(4)]
res["uint8_host_batch"] = rate(lambda n: sc.calculate_coefficients_batch(
    [u8[i % 4] for i in range(n)], [sp] * n))
for name, arr in (("int16_C", m.astype(np.int16) * 3), ("int16_F", np.asfortranarray(m.astype(np.int16))),
                  ("float32_C", m.astype(np.float32)), ("uint8_C_raw", m)):
    pays = [(arr.copy(order="A"), None) for _ in range(4)]
    outs = sc.coefficients_from_payloads(pays[:2], [sp] * 2)
    assert all(o.to_dict() == want for o in outs), name
    res[name] = rate(lambda n: sc.coefficients_from_payloads([pays[i % 4] for i in range(n)], [sp] * n))
    one = sc.coefficients_from_payloads(pays[:1], [sp])[0]
    res[name + "_detail"] = {"h2d_bytes": one.h2d_bytes, "h2d_ms": one.h2d_ms,
                             "host_scan_ms": one.host_scan_ms}
res["int16_over_uint8_time_ratio"] = res["uint8_host_batch"] / res["int16_C"]
print(json.dumps(res, indent=1))
