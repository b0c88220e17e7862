"""Summarise an ncu SASS source-page CSV: hottest instructions and regions by
warp-stall samples (debug helper)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
tot = sum(float(r[iS] or 0) for r in data) or 1.0
print("samples", tot, "instructions", sum(float(r[iE] or 0) for r in data))
W = int(sys.argv[2]) if len(sys.argv) > 2 else 40
win = []
for k in range(0, len(data), W):
    seg = data[k:k + W]
    s = sum(float(r[iS] or 0) for r in seg)
    ops = sorted({r[1].split()[0].split(".")[0] if not r[1].strip().startswith("@")
                  else r[1].split()[1].split(".")[0] for r in seg if r[1].strip()})
    win.append((s, k, " ".join(o for o in ops if o in (
        "MATCH", "ATOMS", "LDG", "STG", "BAR", "LDS", "STS", "SHFL", "DADD", "REDUX", "VOTE",
        "LDL", "STL", "WARPSYNC", "ATOMG", "RED", "POPC", "CALL", "RET"))))
for s, k, t in sorted(win, reverse=True)[:int(sys.argv[3]) if len(sys.argv) > 3 else 15]:
    print(f"{s / tot * 100:5.1f}%  idx {k:5d}  {t}")
print("--- top instructions")
for r in sorted(data, key=lambda r: -float(r[iS] or 0))[:25]:
    print(f"{float(r[iS] or 0) / tot * 100:5.1f}%  {data.index(r):5d} {r[1].strip()[:80]}")

# stall reasons overall and per hot region
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot_r = {c: sum(float(r[h.index(c)] or 0) for r in data) for c in reasons}
print("--- stall reasons (all)")
for c, v in sorted(tot_r.items(), key=lambda x: -x[1])[:8]:
    print(f"  {c:24s} {v / tot * 100:5.1f}%")
if len(sys.argv) > 4:
    for center in map(int, sys.argv[4].split(",")):
        print(f"--- context around {center}")
        for r in data[max(0, center - 12):center + 6]:
            top = max(reasons, key=lambda c: float(r[h.index(c)] or 0))
            print(f"{data.index(r):5d} {float(r[iS] or 0)/tot*100:5.1f}% {top[6:]:14s} {r[1].strip()[:70]}")
