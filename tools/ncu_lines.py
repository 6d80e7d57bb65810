"""Per-source-line breakdown from `ncu -i X --page source --csv --print-source cuda,sass -k K`.

usage: ncu_lines.py <csv> <pixels> [top] [function-substring]
"""
import csv
import io
import sys
from collections import defaultdict


def main(path, npx, top=40, fsub=""):
    fn, fpath, header = "", "", None
    data = defaultdict(lambda: [0.0, 0.0, ""])
    for raw in open(path):
        row = next(csv.reader(io.StringIO(raw)), None)
        if not row:
            continue
        if row[0] == "File Path":
            fpath, header = row[1], None
            continue
        if row[0] == "Function Name":
            fn, header = row[1], None
            continue
        if row[0] == "Line No":
            header = row
            ti = header.index("Thread Instructions Executed")
            wi = header.index("Warp Stall Sampling (All Samples)")
            continue
        if header is None or len(row) <= ti or row[2] != "-" or fsub not in fn:
            continue
        key = (fpath.split("/")[-1], row[0])
        d = data[key]
        d[0] += float(row[ti] or 0)
        d[1] += float(row[wi] or 0)
        d[2] = row[1][:95]
    tot = sum(v[0] for v in data.values())
    tots = sum(v[1] for v in data.values())
    print(f"thread-instr/px {tot / npx:.1f}  stall samples {tots:.0f}")
    col = 1 if __import__("os").environ.get("SORT") == "stall" else 0
    for (f, ln), (v, s, src) in sorted(data.items(), key=lambda kv: -kv[1][col])[:top]:
        print(f"{v / max(tot, 1):6.1%} instr {s / max(tots, 1):6.1%} stall  {f}:{ln:>4} {src}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 40,
         sys.argv[4] if len(sys.argv) > 4 else "")
