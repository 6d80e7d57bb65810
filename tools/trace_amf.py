"""Per-CTA phase timeline of the AMF kernels (needs `make trace`; HYB_LIB=libhybrid_cuda_trace.so).

Slots: k3 kernel 0=start 15=end; growth kernel 0=start 1=counted 2=batch chosen 4=tiles ready
5+l=level l done 14=batch end 15=end.  Prints quantiles (us from the k3 start) over CTAs."""
import ctypes
import os
import sys

os.environ["HYB_LIB"] = "libhybrid_cuda_trace.so"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
from paper_2005_05371_b200 import CONFIGS, capi  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c = CONFIGS[cfg]
g = torch.from_numpy(capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)).cuda()
f = torch.empty_like(g)
ctx = capi.Context(0)
lib = capi.lib
buf = (ctypes.c_ulonglong * (2 * 1024 * 16))()
for rep in range(3):
    lib.hyb_trace_clear()
    torch.cuda.synchronize()
    capi.check(lib.hyb_amf_u8(ctx.ptr, g.data_ptr(), c["cols"], c["rows"], c["cols"], 0, c["rows"], c["smax"],
                              f.data_ptr(), c["cols"], None, c["cols"]), ctx.ptr)
    torch.cuda.synchronize()
lib.hyb_trace_read(buf)
t = np.frombuffer(buf, dtype=np.uint64).reshape(2, 1024, 16).astype(np.int64)
k3, gr = t[0], t[1]
k3 = k3[k3[:, 0] > 0]
gr = gr[gr[:, 15] > 0]
t0 = k3[:, 0].min()


def q(x):
    x = (x - t0) / 1e3
    return " ".join(f"{v:7.2f}" for v in np.percentile(x, [0, 10, 50, 90, 100]))


print(f"config {cfg}: {len(k3)} k3 CTAs, {len(gr)} growth CTAs   quantiles 0/10/50/90/100 (us)")
print("k3 start      ", q(k3[:, 0]))
print("k3 end        ", q(k3[:, 15]))
names = {1: "grow located", 2: "batch chosen", 3: "queue built", 12: "tiles landed", 4: "tiles ready", 14: "batch end", 15: "grow end"}
for s in (1, 2, 3, 12, 4, 5, 6, 7, 8, 14, 15):
    col = gr[:, s]
    col = col[col > 0]
    if len(col):
        print(f"{names.get(s, f'level {2 * (s - 5) + 5} done'):14s}", q(col))
if len(sys.argv) > 2:
    order = np.argsort(-(t[1][:, 2]))[:6]
    for b in order:
        row = t[1][b]
        print("cta", b, " ".join(f"{s}:{(row[s] - t0) / 1e3:.2f}" for s in (1, 9, 10, 11, 2, 3, 12, 4, 5, 6, 15) if row[s] > 0))
