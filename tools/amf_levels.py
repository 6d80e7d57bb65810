"""AMF device time on one BASELINE config for smax = 3, 5, ..., S (marginal cost per growth level)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2005_05371_b200 import CONFIGS, capi  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS[cfg]
g = torch.from_numpy(capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)).cuda()
f = torch.empty_like(g)
ctx = capi.Context(0)
s = torch.cuda.Stream()
ctx.set_stream(s.cuda_stream)
for smax in range(3, c["smax"] + 1, 2):
    def run():
        capi.check(capi.lib.hyb_amf_u8(ctx.ptr, g.data_ptr(), c["cols"], c["rows"], c["cols"], 0, c["rows"], smax,
                                       f.data_ptr(), c["cols"], None, c["cols"]), ctx.ptr)
    for _ in range(3):
        run()
    with torch.cuda.stream(s):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
    torch.cuda.synchronize()
    print(f"config {cfg} smax {smax}: {e0.elapsed_time(e1) / 5 * 1e3:.1f} us")
