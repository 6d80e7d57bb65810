"""Runs hyb_amf_u8 (device buffers) on one BASELINE config a few times -- for ncu launch lists."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2005_05371_b200 import CONFIGS, capi  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = CONFIGS[cfg]
g = torch.from_numpy(capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)).cuda()
f = torch.empty_like(g)
y = torch.empty_like(g)
w = torch.zeros(1, dtype=torch.int64, device="cuda")
ctx = capi.Context(0)
s = torch.cuda.Stream()
ctx.set_stream(s.cuda_stream)
lib = capi.lib
for _ in range(reps):
    capi.check(lib.hyb_amf_u8(ctx.ptr, g.data_ptr(), c["cols"], c["rows"], c["cols"], 0, c["rows"], c["smax"],
                              f.data_ptr(), c["cols"], None, c["cols"]), ctx.ptr)
    w.zero_()
    capi.check(lib.hyb_wiener_stats_u8(ctx.ptr, f.data_ptr(), c["cols"], c["rows"], c["cols"], 0, c["rows"], c["win"],
                                       w.data_ptr()), ctx.ptr)
    capi.check(lib.hyb_wiener_gain_u8(ctx.ptr, f.data_ptr(), c["cols"], c["rows"], c["cols"], 0, c["rows"], c["win"],
                                      w.data_ptr(), c["rows"] * c["cols"], y.data_ptr(), c["cols"]), ctx.ptr)
torch.cuda.synchronize()
print("ok", cfg)
