import csv, sys
lines = open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/lc3.csv').read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.DictReader(lines[start:]))
d = {}
for r in rows:
    key = (int(r['ID']), r['Kernel Name'][:26])
    try:
        d.setdefault(key, {})[r['Metric Name']] = float(r['Metric Value'].replace(',', ''))
    except ValueError:
        pass
items = sorted(d.items())[-14:]
tot = 0
for (i, k), m in items:
    t = m.get('gpu__time_duration.sum', 0) / 1e3
    tot += t
    print(f"{k:26s} {t:7.1f} us  dram {m.get('dram__bytes_read.sum', 0)/1e6:6.1f} MB  L2 {m.get('lts__t_bytes.sum', 0)/1e6:6.1f} MB  "
          f"inst {m.get('smsp__inst_executed.sum', 0)/1e6:5.1f} M  occ {m.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):4.1f} "
          f"issue {m.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):4.1f}")
print("total", round(tot, 1))
