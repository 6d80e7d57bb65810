"""H2D / D2H rate of one config-1 image (2.56 MB) from different pinned host allocations:
torch's pinned allocator, cudaHostRegister'ed numpy memory, and the same first-touched on the current
NUMA node.  usage: pinned_probe.py"""
import ctypes
import time

import numpy as np
import torch

N = 1600 * 1600
dev = torch.empty(N, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()


def rate(h, reps=30):
    res = []
    for direction in ("h2d", "d2h"):
        with torch.cuda.stream(s):
            for _ in range(3):
                (dev.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(dev, non_blocking=True))
            s.synchronize()
            ts = []
            for _ in range(reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                (dev.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(dev, non_blocking=True))
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        res.append(f"{direction} med {ts[len(ts) // 2]:6.1f} us ({N / ts[len(ts) // 2] / 1e3:5.1f} GB/s) min {ts[0]:6.1f}")
    return "  ".join(res)


a = torch.empty(N, dtype=torch.uint8).pin_memory()
print("torch pin_memory()          ", rate(a))
b = torch.empty(N, dtype=torch.uint8, pin_memory=True)
print("torch empty(pin_memory=True)", rate(b))
arr = np.zeros(N + 4096, np.uint8)
off = (-arr.ctypes.data) % 4096
arr2 = arr[off:off + N]
arr2[:] = 1  # first touch
cr = torch.cuda.cudart()
err = cr.cudaHostRegister(arr2.ctypes.data, N, 0)
c = torch.from_numpy(arr2)
print(f"numpy + cudaHostRegister ({int(err)})", rate(c))
big = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
dbig = torch.empty_like(big, device="cuda")
with torch.cuda.stream(s):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dbig.copy_(big, non_blocking=True)
    e0.record()
    for _ in range(5):
        dbig.copy_(big, non_blocking=True)
    e1.record()
    e1.synchronize()
print(f"64 MiB H2D: {5 * big.numel() / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
