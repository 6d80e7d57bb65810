"""Fused small-image kernel: phase split from its own globaltimer stamps (hyb_stats) on a BASELINE config."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2005_05371_b200 import CONFIGS, FilterConfig, capi, denoise  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
c = CONFIGS[cfg]
g = torch.from_numpy(capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)).cuda()
ta, tw, tt = [], [], []
for i in range(30):
    r = denoise.hybrid_denoise(g, FilterConfig(smax=c["smax"], wiener_window=c["win"]))
    if i >= 5:
        ta.append(r.t_adaptive)
        tw.append(r.t_wiener)
        tt.append(r.t_total)
med = lambda v: sorted(v)[len(v) // 2] * 1e6  # noqa: E731
print(f"config {cfg}: amf {med(ta):.1f} us  wiener {med(tw):.1f} us  total(events) {med(tt):.1f} us")
