"""Host-side phase costs of the batch loop (SC_HOST_PROFILE=1), tiny and C2 ROIs."""
import os, sys, time
os.environ["SC_HOST_PROFILE"] = "1"
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2510_02894_b200 as sc
from paper_2510_02894_b200 import _native, synth

tiny = np.zeros((32, 32, 32), np.uint8)
tiny[8:24, 8:24, 8:24] = 1
for name, m, sp in [("tiny", tiny, (1.0, 1.0, 1.0)), ("c2", synth.kits_like(), (0.8, 0.8, 1.0))]:
    d = torch.from_numpy(m).cuda()
    for slots in (1, 8):
        _native.set_option("slots", slots)
        sc.calculate_coefficients_device_batch([d] * 16, [sp] * 16)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sc.calculate_coefficients_device_batch([d] * 200, [sp] * 200)
        torch.cuda.synchronize()
        print(name, "slots", slots, round(200 / (time.perf_counter() - t0)), "ROIs/s", flush=True)
