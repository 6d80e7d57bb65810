"""Copy-engine sequencing probe (2.56 MB pinned): how long an H2D takes depending on what precedes it."""
import numpy as np
import torch

n = 2_560_000
hi = torch.empty(n, dtype=torch.uint8).pin_memory()
ho = torch.empty(n, dtype=torch.uint8).pin_memory()
di = torch.empty(n, dtype=torch.uint8, device="cuda")
do = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
spin = torch.empty(1 << 20, device="cuda")


def run(pattern, trials=60):
    res = {k: [] for k in pattern}
    for _ in range(trials):
        ev = []
        with torch.cuda.stream(s):
            for k in pattern:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record()
                if k == "h2d":
                    di.copy_(hi, non_blocking=True)
                elif k == "d2h":
                    ho.copy_(do, non_blocking=True)
                elif k == "kern":
                    spin.mul_(1.0001)
                ev.append((k, e0))
            e_end = torch.cuda.Event(enable_timing=True)
            e_end.record()
        e_end.synchronize()
        for i, (k, e) in enumerate(ev):
            nxt = ev[i + 1][1] if i + 1 < len(ev) else e_end
            res[k].append(e.elapsed_time(nxt) * 1e3)
    print(" -> ".join(pattern).ljust(32), "  ".join(f"{k} {np.median(v):6.1f}" for k, v in res.items()), "us (median)")


run(["h2d"])
run(["d2h"])
run(["h2d", "d2h"])
run(["h2d", "kern", "d2h"])
run(["d2h", "h2d"])
run(["kern", "h2d", "kern"])
