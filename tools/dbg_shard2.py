import math, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2510_02894_b200 as sc
from paper_2510_02894_b200 import synth
arr = synth.noisy_ellipsoid(512)
got = sc.calculate_coefficients(arr, (1.0, 1.0, 1.0))
d = torch.from_numpy(arr).cuda()
full = sc.calculate_coefficients_device(d, (1.0, 1.0, 1.0)).to_dict()
print("full", full["Maximum3DDiameter"])
sq = torch.zeros(4, dtype=torch.float64, device="cuda")
for n in (2, 4, 8):
    best = torch.zeros(4, dtype=torch.float64, device="cuda")
    for shard in range(n):
        part = sc.calculate_coefficients_shard(d, (1.0, 1.0, 1.0), shard, n, sq)
        torch.maximum(best, sq, out=best)
        print(n, shard, "part", part.max_3d_diameter, "sq", math.sqrt(sq[0].item()), "best", math.sqrt(best[0].item()), flush=True)
