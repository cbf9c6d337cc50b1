"""Batch throughput vs pipeline slots: C2, C5 and a tiny ROI (launch/host floor)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2510_02894_b200 as sc
from paper_2510_02894_b200 import _native, synth

tiny = np.zeros((32, 32, 32), np.uint8)
tiny[8:24, 8:24, 8:24] = 1
cases = [("tiny", tiny, (1.0, 1.0, 1.0)), ("c5", synth.thin_slab(), (0.5, 0.5, 5.0)),
         ("c2", synth.kits_like(), (0.8, 0.8, 1.0))]
for name, m, sp in cases:
    d = torch.from_numpy(m).cuda()
    for graphs in (1, 0):
        _native.set_option("graphs", graphs)
        for slots in (1, 2, 4, 8):
            _native.set_option("slots", slots)
            sc.calculate_coefficients_device_batch([d] * 16, [sp] * 16)
            best = 0
            for rep in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                sc.calculate_coefficients_device_batch([d] * 100, [sp] * 100)
                torch.cuda.synchronize()
                best = max(best, 100 / (time.perf_counter() - t0))
            print(name, "graphs", graphs, "slots", slots, round(best, 1), "ROIs/s", flush=True)
    _native.set_option("graphs", 1)
