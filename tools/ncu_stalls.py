"""Per-kernel stall breakdown from gpurun_out/prof.ncu-rep (source page)."""
import csv, io, subprocess, sys
from collections import Counter

def main(regex, rep="gpurun_out/prof.ncu-rep", top=12):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", f"regex:{regex}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    h = rows[hi]; data = [r for r in rows[hi + 1:] if len(r) == len(h)]
    f = lambda x: float(x) if x.replace('.', '', 1).isdigit() else 0.0
    stalls = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
    tot = {s: sum(f(r[h.index(s)]) for r in data) for s in stalls}
    T = sum(tot.values()) or 1
    print("stalls:", [(s[6:], round(v / T, 3)) for s, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]])
    si = h.index("Source"); a = h.index("Warp Stall Sampling (All Samples)")
    c = Counter()
    for r in data:
        t = r[si].split()
        if t: c[(t[1] if t[0].startswith("@") else t[0]).split(".")[0]] += f(r[a])
    S = sum(c.values()) or 1
    print("by opcode:", [(k, round(v / S, 3)) for k, v in c.most_common(top)])

if __name__ == "__main__":
    main(sys.argv[1])
