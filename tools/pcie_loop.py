"""Mean time of back-to-back [H2D n bytes, D2H n bytes] pairs from pinned memory (the e2e floor)."""
import sys
import time

import torch

n = int(float(sys.argv[1]) * 2**20) if len(sys.argv) > 1 else 2560000
h = torch.empty(n, dtype=torch.uint8).pin_memory()
o = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for mode in ("serial", "serial", "sync-each"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for _ in range(50):
            d.copy_(h, non_blocking=True)
            o.copy_(d, non_blocking=True)
            if mode == "sync-each":
                s.synchronize()
    torch.cuda.synchronize()
    print(f"{mode:10s} {n/1e6:.2f} MB each way: {(time.perf_counter() - t0) / 50 * 1e6:.1f} us per H2D+D2H pair")
