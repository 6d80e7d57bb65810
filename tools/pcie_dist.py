"""Distribution of single H2D / D2H copy times (2.56 MB, pinned) over many trials, for a few host buffers."""
import ctypes
import mmap

import numpy as np
import torch

n = 2_560_000
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
cudart = ctypes.CDLL("libcudart.so")


def dist(h, label, trials=200):
    th, td = [], []
    for _ in range(trials):
        for arr, dst, src in ((th, d, h), (td, h, d)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record()
                dst.copy_(src, non_blocking=True)
                e1.record()
            e1.synchronize()
            arr.append(e0.elapsed_time(e1) * 1e3)
    p = lambda a: " ".join(f"{v:6.1f}" for v in np.percentile(a, [5, 25, 50, 75, 95]))  # noqa: E731
    print(f"{label:28s} h2d us p5/25/50/75/95: {p(th)}   d2h: {p(td)}")


dist(torch.empty(n, dtype=torch.uint8).pin_memory(), "torch pin_memory")
# 2 MiB-aligned anonymous mapping, registered
buf = mmap.mmap(-1, n + (4 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
addr = ctypes.addressof(ctypes.c_char.from_buffer(buf))
al = (addr + (2 << 20) - 1) & ~((2 << 20) - 1)
arr = np.frombuffer(buf, dtype=np.uint8, count=n, offset=al - addr)
arr[:] = 1
rc = cudart.cudaHostRegister(ctypes.c_void_p(al), ctypes.c_size_t(n), 0)
print("cudaHostRegister rc", rc)
dist(torch.from_numpy(arr), "mmap 2MiB-aligned registered")
