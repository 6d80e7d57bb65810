"""Per-source-line profile from `ncu -i X --page source --csv --print-source cuda,sass`: stall samples,
executed warp instructions and the stall-reason mix, summed over the SASS under each source line
(inlined header code is attributed to its own file:line).  usage: ncu_srcprof.py <report> <kernel regex> [top] [launches to skip]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
skip = sys.argv[4] if len(sys.argv) > 4 else "0"  # matching launches to skip (e.g. 1: the second W1 pass)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


fname, hdr, line = "?", None, None
agg = defaultdict(lambda: defaultdict(float))
src = {}
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < len(hdr):
        continue
    if row[0]:
        line = (fname, int(row[0]))
        src[line] = row[1].strip()[:70]
        continue
    if not row[2].startswith("0x"):
        continue
    d = agg[line]
    d["samples"] += num(row[hdr.index("Warp Stall Sampling (All Samples)")])
    d["instr"] += num(row[hdr.index("Instructions Executed")])
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and row[i] not in ("", "0"):
            d[h] += num(row[i])
tot_s = sum(d["samples"] for d in agg.values())
tot_i = sum(d["instr"] for d in agg.values())
print(f"total samples {tot_s:.0f}, warp instructions {tot_i/1e6:.1f} M")
for ln, d in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    st = sorted(((k[6:], v) for k, v in d.items() if k.startswith("stall_")), key=lambda kv: -kv[1])[:4]
    print(f"{ln[0]}:{ln[1]:5d} {100*d['samples']/tot_s:5.1f}% smp {100*d['instr']/tot_i:5.1f}% ins  "
          + " ".join(f"{k}={100*v/max(d['samples'],1):.0f}" for k, v in st) + f"  | {src.get(ln, '')}")
