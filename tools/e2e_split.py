"""Host-buffer hybrid call split: H2D (upload) vs kernel time from hyb_stats, and the wall time per call."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2005_05371_b200 import CONFIGS, capi  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c = CONFIGS[cfg]
rows, cols = c["rows"], c["cols"]
h = torch.from_numpy(capi.make_phantom(rows, cols, c["ellipses"], c["sigma"], c["density"], 0)).pin_memory()
o = torch.empty_like(h).pin_memory()
ctx = capi.Context(0)
st = capi.HybStats()
tot, amf, wie, wall = [], [], [], []
for i in range(40):
    t0 = time.perf_counter()
    capi.check(capi.lib.hyb_hybrid_u8(ctx.ptr, h.data_ptr(), cols, rows, cols, c["smax"], c["win"], 1, o.data_ptr(),
                                      cols, ctypes.byref(st)), ctx.ptr)
    wall.append(time.perf_counter() - t0)
    if i >= 5:
        tot.append(st.t_total)
        amf.append(st.t_adaptive)
        wie.append(st.t_wiener)
med = lambda v: sorted(v)[len(v) // 2] * 1e6  # noqa: E731
print(f"config {cfg}: upload+kernel {med(tot):.1f} us (kernel amf {med(amf):.1f} + wiener {med(wie):.1f}); "
      f"wall per call {med(wall[5:]):.1f} us")

# same step with torch doing the copies around the device-buffer call, for comparison
dg = torch.empty_like(h, device="cuda")
dy = torch.empty_like(dg)
s = torch.cuda.Stream()
ctx.set_stream(s.cuda_stream)
ts = []
for i in range(40):
    with torch.cuda.stream(s):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        dg.copy_(h, non_blocking=True)
        e1.record()
        capi.check(capi.lib.hyb_hybrid_u8(ctx.ptr, dg.data_ptr(), cols, rows, cols, c["smax"], c["win"], 1,
                                          dy.data_ptr(), cols, None), ctx.ptr)
        o.copy_(dy, non_blocking=True)
        e2.record()
    e2.synchronize()
    if i >= 5:
        ts.append((e0.elapsed_time(e1) * 1e3, e1.elapsed_time(e2) * 1e3))
ts.sort(key=lambda t: t[0] + t[1])
print(f"torch copies: h2d {ts[len(ts) // 2][0]:.1f} us, kernel + d2h {ts[len(ts) // 2][1]:.1f} us")
