"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel."""
import csv
import sys
from collections import defaultdict


def summarise(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr, rows = rows[0], rows[1:]
    ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
    d = defaultdict(list)
    for r in rows:
        d[(r[ki].split("(")[0], r[gi])].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    out = []
    for (k, g), v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"{k:55s} grid={g:14s} n={len(v):4d} avg={sum(v)/len(v)/1e3:9.2f} us share={sum(v)/tot:6.1%}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
