"""Runs hyb_hybrid_batch_u8 on device buffers for the config-3 stack (512 slices of 512^2), for ncu
captures.  usage: batch_dev.py [slices] [reps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2005_05371_b200 import CONFIGS, capi  # noqa: E402

c = CONFIGS[3]
n = int(sys.argv[1]) if len(sys.argv) > 1 else c["slices"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rows, cols = c["rows"], c["cols"]
host = np.stack([capi.make_phantom(rows, cols, c["ellipses"], c["sigma"], c["density"], s) for s in range(n)])
g = torch.from_numpy(host).cuda()
y = torch.empty_like(g)
ctx = capi.Context(0)
for _ in range(reps):
    capi.check(capi.lib.hyb_hybrid_batch_u8(ctx.ptr, g.data_ptr(), cols, rows * cols, n, rows, cols, c["smax"],
                                            c["win"], y.data_ptr(), cols, rows * cols, None), ctx.ptr)
torch.cuda.synchronize()
print("ok config 3", n)
