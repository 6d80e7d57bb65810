"""Per-CTA phase timeline of the fused small-image kernel (needs `make trace`)."""
import ctypes
import os
import sys

os.environ.setdefault("HYB_LIB", "libhybrid_cuda_trace.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
from paper_2005_05371_b200 import CONFIGS, FilterConfig, capi, denoise  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c = CONFIGS[cfg]
g = torch.from_numpy(capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)).cuda()
y = torch.empty_like(g)
ctx = capi.Context(0)
for _ in range(5):
    capi.check(capi.lib.hyb_hybrid_u8(ctx.ptr, g.data_ptr(), c["cols"], c["rows"], c["cols"], c["smax"], c["win"], 1,
                                      y.data_ptr(), c["cols"], None), ctx.ptr)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (2 * 1024 * 16))()
capi.lib.hyb_trace_read_small(buf)
t = np.frombuffer(buf, dtype=np.uint64).reshape(2, 1024, 16).astype(np.int64)[0]
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
names = ["start", "g landed", "edges", "k=3 done", "queue", "growth done", "own stats", "barrier 1", "f landed",
         "f edges", "stats done", "barrier 2", "gain done"]
slots = [0, 1, 2, 3, 4, 5, 14, 6, 7, 8, 9, 10, 11]
print(f"config {cfg}: {len(t)} CTAs   quantiles 0/10/50/90/100 (us)")
for s, nm in zip(slots, names):
    if not t[:, s].any():
        continue
    col = (t[:, s] - t0) / 1e3
    print(f"{nm:12s}", " ".join(f"{v:7.2f}" for v in np.percentile(col, [0, 10, 50, 90, 100])))

order = np.argsort(-t[:, 5])[:12]
print("slowest growth CTAs: tiles failures | edges k3done queue growth (us)")
for b in order:
    r = t[b]
    print(f"  tiles {r[13]} failures {r[12]:5d} |", " ".join(f"{(r[s] - t0) / 1e3:6.2f}" for s in (2, 3, 4, 5)))
fl = t[:, 12]
print("failures per CTA: min/median/max", fl.min(), int(np.median(fl)), fl.max())
