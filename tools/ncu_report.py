"""Text summary of an `ncu --set full` report: per kernel launch, the metrics the roofline and
the DESIGN.md analysis use.  usage: ncu_report.py <file.ncu-rep> [pixels]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration_us", 1e-3),
    ("dram__bytes_read.sum", "dram_read_MB", 1.0),
    ("dram__bytes_write.sum", "dram_write_MB", 1.0),
    ("smsp__inst_executed.sum", "warp_instr_M", 1e-6),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%", 1.0),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pipe_%", 1.0),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%", 1.0),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_pipe_%", 1.0),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_pipe_%", 1.0),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%", 1.0),
    ("launch__registers_per_thread", "regs", 1.0),
]


def main(path, pixels=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {k: hdr.index(k) for k, _, _ in KEYS if k in hdr}
    ki = hdr.index("Kernel Name")
    print("kernel".ljust(46) + "".join(n.rjust(15) for _, n, _ in KEYS))
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "").replace("hyb::<unnamed>::", "")[:45]
        vals = []
        for k, n, sc in KEYS:
            if k not in idx:
                vals.append("-")
                continue
            v = float(r[idx[k]].replace(",", "") or 0)
            u = units[idx[k]]
            if k.startswith("dram__bytes"):
                v = v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "B": 1e-6, "KB": 1e-3, "MB": 1.0, "GB": 1e3}.get(u, 1.0)
            elif k == "gpu__time_duration.sum":
                v = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
            else:
                v *= sc
            vals.append(f"{v:.2f}")
        print(name.ljust(46) + "".join(v.rjust(15) for v in vals))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
