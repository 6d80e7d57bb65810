"""Runs hyb_hybrid_u8 on device buffers for one BASELINE config (for ncu captures / launch lists)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2005_05371_b200 import CONFIGS, capi  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = CONFIGS[cfg]
g = torch.from_numpy(capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)).cuda()
y = torch.empty_like(g)
ctx = capi.Context(0)
for _ in range(reps):
    capi.check(capi.lib.hyb_hybrid_u8(ctx.ptr, g.data_ptr(), c["cols"], c["rows"], c["cols"], c["smax"], c["win"], 1,
                                      y.data_ptr(), c["cols"], None), ctx.ptr)
torch.cuda.synchronize()
print("ok", cfg)
