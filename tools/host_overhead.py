"""Host-side cost of one hyb_hybrid_u8 call (device buffers, graph replay) vs the device time per step."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2005_05371_b200 import CONFIGS, capi  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c = CONFIGS[cfg]
g = torch.from_numpy(capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)).cuda()
y = torch.empty_like(g)
ctx = capi.Context(0)
s = torch.cuda.Stream()
ctx.set_stream(s.cuda_stream)
lib = capi.lib
args = (ctx.ptr, g.data_ptr(), c["cols"], c["rows"], c["cols"], c["smax"], c["win"], 1, y.data_ptr(), c["cols"], None)
for _ in range(10):
    lib.hyb_hybrid_u8(*args)
torch.cuda.synchronize()
n = 500
t0 = time.perf_counter()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    e0.record()
    for _ in range(n):
        lib.hyb_hybrid_u8(*args)
    t_host = time.perf_counter() - t0
    e1.record()
torch.cuda.synchronize()
t_all = time.perf_counter() - t0
print(f"config {cfg}: host issue {t_host / n * 1e6:.1f} us/call, device {e0.elapsed_time(e1) / n * 1e3:.1f} us/step, "
      f"wall {t_all / n * 1e6:.1f} us/step")
