"""H2D / D2H time vs transfer size from pinned host memory (CUDA events, best of 10)."""
import torch

for mb in (0.0625, 0.25, 1, 2.5, 4, 16, 64):
    n = int(mb * 2**20)
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    res = []
    for direction in ("h2d", "d2h"):
        best = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if direction == "h2d":
                d.copy_(h, non_blocking=True)
            else:
                h.copy_(d, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3)
        res.append(f"{direction} {best:8.1f} us {n / best / 1e3:6.1f} GB/s")
    print(f"{mb:8.3f} MB: " + "   ".join(res))
