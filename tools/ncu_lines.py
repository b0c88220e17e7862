"""Per-source-line totals (instructions executed, stall samples, shared
wavefronts) from `ncu -i X --page source --csv --print-source cuda,sass`
(profiling helper)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
agg = defaultdict(lambda: [0.0, 0.0, 0.0])
src = {}
f = None
h = None
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = r
        iE = h.index("Instructions Executed")
        iS = h.index("Warp Stall Sampling (All Samples)")
        iW = h.index("L1 Wavefronts Shared")
        continue
    if h is None or len(r) < len(h):
        continue
    if r[0].strip():
        line = (f, int(r[0]))
        src[line] = r[1].strip()
    if line is None or not r[2].strip():
        continue
    a = agg[line]
    num = lambda x: float(x) if x.replace(".", "").replace("e+", "").isdigit() else 0.0
    a[0] += num(r[iE])
    a[1] += num(r[iS])
    a[2] += num(r[iW])
tot = [sum(v[k] for v in agg.values()) or 1 for k in range(3)]
print(f"total inst {tot[0]:.3e} stall samples {tot[1]:.0f} smem wavefronts {tot[2]:.3e}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50
key = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = sorted(agg.items(), key=lambda kv: -kv[1][key])[:n]
for (fl, ln), v in sorted(top):
    print(f"{fl:18s}{ln:5d} inst {v[0]/tot[0]*100:5.1f}% stall {v[1]/tot[1]*100:5.1f}% wf {v[2]/tot[2]*100:5.1f}%  {src.get((fl, ln), '')[:70]}")
