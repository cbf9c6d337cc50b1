"""Host-side probe for the host_crop path: slab-scan time vs host threads on
the C2 mask, and pinned H2D bandwidth (torch copy, for comparison)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_2510_02894_b200 import _native, synth  # noqa: E402

m = synth.kits_like(512, 512, 600, (0.8, 0.8, 1.0), 30.0)
pm = torch.from_numpy(m).pin_memory()
arr = pm.numpy()
print("cpu_count", os.cpu_count(), "slab", _native.occupied_slab(arr))
for t in (1, 2, 4, 8, 12, 16, 24, 32, 64):
    if t > (os.cpu_count() or 1):
        break
    _native.occupied_slab(arr, threads=t)
    ts = []
    for _ in range(7):
        t0 = time.perf_counter()
        _native.occupied_slab(arr, threads=t)
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"threads {t:3d}: scan {ts[3]*1e3:.3f} ms  ({m.size / ts[3] / 1e9:.1f} GB/s of mask)")
d = torch.empty(m.size, dtype=torch.uint8, device="cuda")
flat = pm.view(-1)
for _ in range(3):
    d.copy_(flat, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    d.copy_(flat, non_blocking=True)
e1.record()
torch.cuda.synchronize()
print(f"pinned H2D: {10 * m.size / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")
