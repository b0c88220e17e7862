"""Kernel launch list (name, grid, block, duration ns) from an ncu
`--metrics gpu__time_duration.sum --csv` log (profiling helper)."""
import csv
import sys


def rows(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rd = csv.reader(lines)
    hdr = next(rd)
    iN, iG, iB, iV = (hdr.index(k) for k in ("Kernel Name", "Grid Size", "Block Size", "Metric Value"))
    for r in rd:
        yield r[iN], r[iG], r[iB], float(r[iV].replace(",", ""))


if __name__ == "__main__":
    for name, g, b, v in rows(sys.argv[1]):
        print(f"{v / 1e3:9.1f} us  {g:>16s} {b:>14s}  {name[:110]}")
