import sys, time
sys.path.insert(0, '.')
import torch
import paper_2510_02894_b200 as sc
from paper_2510_02894_b200 import _native, synth
w = sys.argv[1] if len(sys.argv) > 1 else "c5"
m, sp = (synth.thin_slab(), (0.5, 0.5, 5.0)) if w == "c5" else (synth.kits_like(), (0.8, 0.8, 1.0))
d = torch.from_numpy(m).cuda()
s = torch.cuda.Stream()
for graphs in (1, 0):
    _native.set_option("graphs", graphs)
    for K in (3, 30, 30, 100):
        for use_stream in (True, False):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            outs = sc.calculate_coefficients_device_batch([d] * K, [sp] * K, stream=s if use_stream else None)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            tot = [round(o.total_ms, 3) for o in outs[:6]]
            print(f"graphs={graphs} K={K} stream={use_stream} {K/dt:.1f} ROIs/s  first totals {tot} mesh {outs[-1].mesh_ms:.3f} diam {outs[-1].diameters_ms:.3f}")
    t0 = time.perf_counter()
    for _ in range(30):
        c = sc.calculate_coefficients_device(d, sp)
    torch.cuda.synchronize()
    print("single", 30 / (time.perf_counter() - t0))
