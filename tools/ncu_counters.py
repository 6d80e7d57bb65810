"""Per-launch DRAM bytes and warp instructions of each stage from an `ncu --set full` report ->
profiles/ncu_counters.json (read by bench.py).  usage: ncu_counters.py <config> <file.ncu-rep>
Stages: hybrid_small_kernel (fused), amf (k3 + growth, or the fused per-batch AMF kernel), wiener (statistics + gain); launches of a
stage are summed (one hybrid call)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNITS = {"byte": 1, "B": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}


def stage(name):
    if "hybrid_small" in name:
        return "hybrid_small_kernel"
    if "amf_k3" in name or "amf_grow" in name or "amf_fused" in name:
        return "amf"
    if "wiener" in name:
        return "wiener"
    return None


def main(cfg, rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki, ri, wi = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    ii = hdr.index("smsp__inst_executed.sum")
    out = {}
    for r in data:
        st = stage(r[ki])
        if not st:
            continue
        b = float(r[ri].replace(",", "")) * UNITS.get(units[ri], 1) + float(r[wi].replace(",", "")) * UNITS.get(units[wi], 1)
        n = float(r[ii].replace(",", ""))
        d = out.setdefault(st, {"dram_bytes": 0, "warp_instr": 0})
        d["dram_bytes"] += int(b)
        d["warp_instr"] += int(n)
    path = os.path.join(ROOT, "profiles", "ncu_counters.json")
    allc = json.load(open(path)) if os.path.exists(path) else {}
    allc[f"config{cfg}"] = out
    allc["_source"] = ("ncu --set full --clock-control none captures of python tools/hybrid_dev.py <config> "
                       "(per-launch dram__bytes_read.sum + dram__bytes_write.sum, smsp__inst_executed.sum)")
    json.dump(allc, open(path, "w"), indent=1, sort_keys=True)
    print(cfg, out)


if __name__ == "__main__":
    main(int(sys.argv[1]), sys.argv[2])
