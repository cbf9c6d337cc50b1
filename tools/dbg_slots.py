import sys, time
sys.path.insert(0, '.')
import torch
import paper_2510_02894_b200 as sc
from paper_2510_02894_b200 import _native, synth
for name, m, sp in (("c2", synth.kits_like(), (0.8, 0.8, 1.0)), ("c5", synth.thin_slab(), (0.5, 0.5, 5.0))):
    d = torch.from_numpy(m).cuda()
    for slots in (2, 4, 6, 8):
        _native.set_option("slots", slots)
        sc.calculate_coefficients_device_batch([d] * 8, [sp] * 8)
        best = 0
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sc.calculate_coefficients_device_batch([d] * 60, [sp] * 60)
            torch.cuda.synchronize()
            best = max(best, 60 / (time.perf_counter() - t0))
        print(name, "slots", slots, round(best, 1), "ROIs/s")
