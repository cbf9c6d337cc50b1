"""A few single-ROI calls (C2) for ncu captures: no probes, no batch overlap."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2510_02894_b200 as sc
from paper_2510_02894_b200 import synth

d = torch.from_numpy(synth.kits_like()).cuda()
for _ in range(3):
    c = sc.calculate_coefficients_device(d, (0.8, 0.8, 1.0))
torch.cuda.synchronize()
print(c.to_dict())
