"""Per-CUDA-source-line instruction counts and stall samples of one kernel in an
ncu report (source page, cuda,sass view; needs -lineinfo + --import-source).

usage: python tools/ncu_lines.py <report> <kernel-regex> [top]"""
import csv
import subprocess
import sys

rep, k = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{k}",
                      "--launch-count", "1", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


lines, cur, fname = [], None, ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0]:  # a source line row (aggregated)
        cur = (fname, r[0], r[1].strip())
        lines.append([cur, num(r[7]), num(r[6])])
tot_i = sum(x[1] for x in lines) or 1
tot_s = sum(x[2] for x in lines) or 1
print(f"{k}: {tot_i:.0f} warp instructions, {tot_s:.0f} samples")
for (f, ln, src), ins, smp in sorted(lines, key=lambda x: -x[1])[:top]:
    print(f"{f}:{ln:>4} inst {ins / tot_i:6.1%} smp {smp / tot_s:6.1%}  {src[:90]}")
