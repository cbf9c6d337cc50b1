"""Summarise an ncu capture + launch list into profiles/ (committed evidence).

usage: python tools/ncu_summary.py <tag>   (reads gpurun_out/prof.ncu-rep and
gpurun_out/launches.csv; writes profiles/ncu_<tag>.md, profiles/ncu_summary.json)
"""

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "pipe_fma_pct"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "pipe_alu_pct"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "inst_fma_pct"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "pipe_fp64_pct"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "s": 1.0, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def short(name):
    name = name.split("(")[0]
    return name.replace("void ", "").split("<")[0].strip()


def raw():
    rep = os.path.join(OUT, "prof.ncu-rep")
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units, data = rows[0], rows[1], rows[2:]
    out = defaultdict(list)
    for r in data:
        k = short(r[h.index("Kernel Name")])
        rec = {}
        for m, alias in METRICS:
            if m in h:
                i = h.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                rec[alias] = v * SCALE.get(units[i], 1)
        out[k].append(rec)
    return out


def launches():
    path = os.path.join(OUT, "launches.csv")
    if not os.path.exists(path):
        return {}
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        try:
            agg[short(r[h.index("Kernel Name")])].append(float(r[h.index("Metric Value")]
                                                               .replace(",", "")))
        except (ValueError, IndexError):
            pass
    return {k: {"n": len(v), "mean_ns": sum(v) / len(v)} for k, v in agg.items()}


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    full = raw()
    lst = launches()
    summ = {"tag": tag, "dram_bytes_per_launch": {}, "kernels": {}}
    lines = [f"# ncu summary {tag}", "",
             "Captured with `ncu --set full --clock-control none` under gpurun (1 B200); "
             "values are per launch (mean over captured launches).", "",
             "| kernel | time us | DRAM rd MB | DRAM wr MB | DRAM % | issue % | FMA pipe % | "
             "ALU pipe % | FP64 pipe % | occupancy % | regs |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for k, recs in full.items():
        avg = {a: sum(r.get(a, 0) for r in recs) / len(recs) for _, a in METRICS}
        summ["kernels"][k] = avg
        summ["dram_bytes_per_launch"][k] = avg["dram_read"] + avg["dram_write"]
        lines.append(f"| {k} | {avg['time'] * 1e6:.1f} | {avg['dram_read'] / 1e6:.2f} | "
                     f"{avg['dram_write'] / 1e6:.2f} | {avg['dram_pct']:.1f} | {avg['issue_pct']:.1f} | "
                     f"{avg['pipe_fma_pct']:.1f} | {avg['pipe_alu_pct']:.1f} | "
                     f"{avg['pipe_fp64_pct']:.1f} | {avg['occupancy_pct']:.1f} | {avg['regs']:.0f} |")
    if lst:
        tot = sum(v["mean_ns"] for k, v in lst.items() if "probe" not in k)
        lines += ["", "Launch list (`--metrics gpu__time_duration.sum`, cold, serialised):", "",
                  "| kernel | launches | mean us | share of ROI |", "|---|---|---|---|"]
        for k, v in sorted(lst.items(), key=lambda kv: -kv[1]["mean_ns"]):
            share = "" if "probe" in k else f"{v['mean_ns'] / tot:.3f}"
            lines.append(f"| {k} | {v['n']} | {v['mean_ns'] / 1e3:.1f} | {share} |")
        summ["launch_list"] = lst
    open(os.path.join(PROF, f"ncu_{tag}.md"), "w").write("\n".join(lines) + "\n")
    json.dump(summ, open(os.path.join(PROF, "ncu_summary.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
