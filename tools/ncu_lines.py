"""Per-source-line breakdown from `ncu -i X --page source --csv --print-source cuda,sass -k K`."""
import csv
import sys


def main(path, npx, top=40):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    h = rows[hi]
    ti = h.index("Thread Instructions Executed")
    wi = h.index("Warp Stall Sampling (All Samples)")
    ie = h.index("Instructions Executed")
    data, tot, totw, tots = [], 0.0, 0.0, 0.0
    for r in rows[hi + 1:]:
        if len(r) <= ti or r[2] != "-":
            continue  # only the per-CUDA-line aggregate rows (Address == "-")
        v, s, w = float(r[ti] or 0), float(r[wi] or 0), float(r[ie] or 0)
        tot += v
        tots += s
        totw += w
        data.append((v, s, r[0], r[1][:100]))
    print(f"thread-instr/px {tot / npx:.1f}  warp-instr total {totw:.3g}  stall samples {tots:.0f}")
    for v, s, ln, src in sorted(data, reverse=True)[:top]:
        print(f"{v / tot:6.1%} instr {s / max(tots, 1):6.1%} stall  L{ln:>4} {src}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 40)
