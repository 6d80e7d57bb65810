"""Phase profile of the fast growth levels (zero / 255 bit planes; needs `make trace`): per CTA, the summed
time of each batch phase and of each level interval.  usage: trace_fast.py [config]"""
import ctypes
import os
import sys

os.environ.setdefault("HYB_LIB", "libhybrid_cuda_trace.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
from paper_2005_05371_b200 import CONFIGS, capi  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS[cfg]
g = torch.from_numpy(capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)).cuda()
f = torch.empty_like(g)
ctx = capi.Context(0)
lib = capi.lib
buf = (ctypes.c_ulonglong * (2 * 1024 * 16))()
for rep in range(2):
    lib.hyb_trace_clear()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    capi.check(lib.hyb_amf_u8(ctx.ptr, g.data_ptr(), c["cols"], c["rows"], c["cols"], 0, c["rows"], c["smax"],
                              f.data_ptr(), c["cols"], None, c["cols"]), ctx.ptr)
    e1.record()
    torch.cuda.synchronize()
lib.hyb_trace_read(buf)
tt = np.frombuffer(buf, dtype=np.uint64).reshape(2, 1024, 16).astype(np.int64)
t = tt[1]
t = t[(t[:, 4] > 0)]
print(f"config {cfg}: AMF call {e0.elapsed_time(e1) * 1e3:.1f} us, {len(t)} growth CTAs, batches/CTA {t[:, 4].mean():.1f}")
names = {13: "entry", 1: "promote + loads issued", 3: "tile wait + edges", 9: "planes",
         11: "dense k=5 + queue build", 5: "B(5) | A(7)", 6: "B(7) | A(9 -> 11)", 7: "B(9) | B(11)", 8: "flagged leftovers"}
tot = 0.0
for s in (13, 1, 3, 9, 11, 5, 6, 7, 8):
    v = t[:, s] / 1e3
    tot += v.mean()
    print(f"{names[s]:24s} per-CTA mean {v.mean():8.1f} us   max {v.max():8.1f}   per batch {1e3 * v.mean() / t[:, 4].mean():7.0f} ns")
print(f"sum of means {tot:.1f} us")
k3s = tt[0][:, 0][tt[0][:, 0] > 0]
ge = tt[1][:, 15][tt[1][:, 15] > 0]
if len(k3s) and len(ge):
    t0 = k3s.min()
    print("growth end, us from the k3 start, quantiles 0/10/50/90/100:",
          " ".join(f"{x:8.1f}" for x in np.percentile((ge - t0) / 1e3, [0, 10, 50, 90, 100])))
