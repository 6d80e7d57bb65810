"""Growth-level profile of the AMF growth kernel (needs `make trace`): per CTA, the summed time spent in
each level k = 5, 7, 9, 11 and the pixels it processed.  usage: trace_levels.py [config]"""
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
t = np.frombuffer(buf, dtype=np.uint64).reshape(2, 1024, 16).astype(np.int64)[1]
t = t[(t[:, 5] > 0)]
print(f"config {cfg}: AMF call {e0.elapsed_time(e1) * 1e3:.1f} us, {len(t)} growth CTAs")
for l, k in enumerate(range(5, c["smax"] + 1, 2)):
    tm, px = t[:, 5 + l] / 1e3, t[:, 9 + l]
    print(f"k={k:2d}: per-CTA level time mean {tm.mean():8.1f} us  max {tm.max():8.1f}   pixels/CTA mean {px.mean():9.0f}"
          f"   ns/pixel/CTA {1e3 * tm.sum() / max(1, px.sum()):7.2f}")
tot = sum(t[:, 5 + l] for l in range(4)) / 1e3
print(f"batches/CTA mean {t[:, 4].mean():.1f}; per CTA mean us: entry {t[:, 13].mean() / 1e3:.1f}  choose {t[:, 1].mean() / 1e3:.1f}"
      f"  queue {t[:, 2].mean() / 1e3:.1f}  wait+edges {t[:, 3].mean() / 1e3:.1f}  levels {tot.mean():.1f}")
print(f"queue detail (warp 0, per CTA us): bitmap load + scan {t[:, 0].mean() / 1e3:.1f}  emission {t[:, 14].mean() / 1e3:.1f}")
tt = np.frombuffer(buf, dtype=np.uint64).reshape(2, 1024, 16).astype(np.int64)
k3s = tt[0][:, 0][tt[0][:, 0] > 0]
k3e = tt[0][:, 15][tt[0][:, 15] > 0]
ge = tt[1][:, 15][tt[1][:, 15] > 0]
t0 = k3s.min()
q = lambda v: " ".join(f"{x:8.1f}" for x in np.percentile((v - t0) / 1e3, [0, 10, 50, 90, 100]))
print("us from the k3 start, quantiles 0/10/50/90/100 over CTAs")
print("k3 end     ", q(k3e))
print("growth end ", q(ge))
