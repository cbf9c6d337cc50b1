"""Per-kernel SM-time census from an ncu CSV (tools/batch_cost.py capture):
duration, warps resident x time (sm__warps_active.sum / clock), instructions.
usage: ncu_cost.py <csv> [n_rois]"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
ii = h.index("ID")
per = defaultdict(dict)
names = {}
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    per[r[ii]][r[mi]] = (v, r[ui])
    names[r[ii]] = r[ki].split("(")[0].replace("void ", "").split("<")[0].strip()
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    t, tu = m.get("gpu__time_duration.sum", (0, "ns"))
    t_us = t / 1e3 if tu == "ns" else t * (1e3 if tu == "ms" else 1)
    clk = m.get("sm__cycles_elapsed.avg.per_second", (1.9e9, "hz"))[0]
    clk = clk * {"hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}.get(m.get("sm__cycles_elapsed.avg.per_second", (0, "Ghz"))[1], 1)
    wa = m.get("sm__warps_active.sum", (0, ""))[0]
    a[0] += 1
    a[1] += t_us
    a[2] += wa / clk * 1e6  # warp-us
    a[3] += m.get("smsp__inst_executed.sum", (0, ""))[0]
    a[4] += m.get("launch__grid_size", (0, ""))[0]
tot = sum(a[2] for a in agg.values())
print(f"{'kernel':18s} {'launch':>6s} {'us/ROI':>8s} {'warp-us/ROI':>12s} {'share':>6s} {'Minst/ROI':>9s} {'grid':>6s}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][2]):
    print(f"{k:18s} {a[0]:6d} {a[1] / n:8.2f} {a[2] / n:12.0f} {a[2] / tot:6.3f} {a[3] / n / 1e6:9.3f} {a[4] / a[0]:6.0f}")
print(f"total warp-us/ROI {tot / n:.0f}  (GPU capacity: 148 SMs x 64 warps = 9472 warps -> "
      f"{tot / n / 9472:.2f} us/ROI if every warp slot were busy)")
