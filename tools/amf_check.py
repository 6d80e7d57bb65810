"""Full-size AMF parity spot check: GPU hyb_amf_u8 vs the C oracle on one BASELINE config
(optionally a row crop / another smax).  usage: amf_check.py <config> [rows] [repeats] [smax]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2005_05371_b200 import CONFIGS, capi  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CONFIGS[cfg]
rows = int(sys.argv[2]) if len(sys.argv) > 2 else c["rows"]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
if len(sys.argv) > 4:
    c = dict(c, smax=int(sys.argv[4]))
g = capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)[:rows].copy()
want, wfin = oracle.amf(g, c["smax"], finalized_at=True)
gd = torch.from_numpy(g).cuda()
f = torch.empty_like(gd)
ctx = capi.Context(0)
for r in range(reps):
    f.fill_(7)
    torch.cuda.synchronize()
    capi.check(capi.lib.hyb_amf_u8(ctx.ptr, gd.data_ptr(), c["cols"], rows, c["cols"], 0, rows, c["smax"],
                                   f.data_ptr(), c["cols"], None, c["cols"]), ctx.ptr)
    torch.cuda.synchronize()  # the context runs on its own (non-blocking) stream
    got = f.cpu().numpy()
    bad = int((got != want).sum())
    print(f"config {cfg} rows {rows} rep {r}: mismatches {bad}")
    if bad:
        ys, xs = np.nonzero(got != want)
        lv, cnt = np.unique(wfin[ys, xs], return_counts=True)
        tiles = np.unique((ys // 32) * 1000 + xs // 128)
        print("  rows%32:", np.bincount(ys % 32, minlength=32).tolist(), " cols%128 min/max:", int((xs % 128).min()), int((xs % 128).max()))
        print("  got/want sample:", [(int(y), int(x), int(got[y, x]), int(want[y, x]), int(g[y, x])) for y, x in zip(ys[:8], xs[:8])])
        print("  by oracle level:", dict(zip(lv.tolist(), cnt.tolist())), "tiles:", len(tiles), tiles[:12].tolist())
