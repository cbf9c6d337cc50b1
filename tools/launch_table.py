"""Print the per-kernel times of the last ROI in ncu launch lists (gpurun_out/launches_<w>.csv)."""
import csv
import sys

for w in sys.argv[1:] or ["c2", "c3"]:
    path = f"gpurun_out/launches_{w}.csv"
    rows = list(csv.DictReader(l for l in open(path) if not l.startswith("==")))
    ks = [(r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", ""), float(r["Metric Value"]))
          for r in rows if r["Metric Name"] == "gpu__time_duration.sum"]
    start = max(i for i, (k, _) in enumerate(ks) if k == "init_stats")
    last = ks[start:]
    print(f"{w}: {len(last)} kernels, total {sum(v for _, v in last) / 1e3:.1f} us (cold, serialised)")
    for k, v in last:
        print(f"  {k:22s} {v / 1e3:9.1f} us")
