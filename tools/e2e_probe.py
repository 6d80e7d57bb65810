"""Breaks down the end-to-end (host-buffer) hybrid call: raw pinned copy bandwidth vs API time."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2005_05371_b200 import CONFIGS, capi  # noqa: E402

c = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
rows, cols = c["rows"], c["cols"]
h = torch.from_numpy(capi.make_phantom(rows, cols, c["ellipses"], c["sigma"], c["density"], 0)).pin_memory()
o = torch.empty_like(h).pin_memory()
d = torch.empty_like(h, device="cuda")
s = torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record()
    for _ in range(20):
        d.copy_(h, non_blocking=True)
    e1.record()
torch.cuda.synchronize()
print(f"H2D {h.numel() * 20 / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
with torch.cuda.stream(s):
    e0.record()
    for _ in range(20):
        o.copy_(d, non_blocking=True)
    e1.record()
torch.cuda.synchronize()
print(f"D2H {h.numel() * 20 / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
ctx = capi.Context(0)
st = capi.HybStats()
for i in range(5):
    capi.check(capi.lib.hyb_hybrid_u8(ctx.ptr, h.data_ptr(), cols, rows, cols, c["smax"], c["win"], 1, o.data_ptr(),
                                      cols, ctypes.byref(st)), ctx.ptr)
t0 = time.perf_counter()
n = 20
for i in range(n):
    capi.check(capi.lib.hyb_hybrid_u8(ctx.ptr, h.data_ptr(), cols, rows, cols, c["smax"], c["win"], 1, o.data_ptr(),
                                      cols, ctypes.byref(st)), ctx.ptr)
wall = (time.perf_counter() - t0) / n
print(f"api wall {wall * 1e6:.1f} us; device: amf {st.t_adaptive * 1e6:.1f} wiener {st.t_wiener * 1e6:.1f} "
      f"total(incl copies) {st.t_total * 1e6:.1f} us")
t0 = time.perf_counter()
for i in range(n):
    capi.check(capi.lib.hyb_hybrid_u8(ctx.ptr, h.data_ptr(), cols, rows, cols, c["smax"], c["win"], 1, o.data_ptr(),
                                      cols, None), ctx.ptr)
print(f"api wall without stats {(time.perf_counter() - t0) / n * 1e6:.1f} us")
