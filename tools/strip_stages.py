"""Stage split of one strip of the multi-GPU step on one GPU (CUDA events, warm): AMF, W1 statistics, W1
gain for N = 1 / 2 / 4 / 8 strips (every rank), to see which stage loses efficiency as strips shrink.
usage: strip_stages.py [config]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2005_05371_b200 import CONFIGS, capi  # noqa: E402
from paper_2005_05371_b200.partition import CudaStripBackend, StripPlan  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS[cfg]
ctx = capi.Context(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx.set_stream(s.cuda_stream)
be = CudaStripBackend(ctx)
g_full = torch.from_numpy(capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)).cuda()


def timed(fn, k=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3


ranks_of = {1: [0], 2: [0, 1], 4: [0, 1, 2, 3], 8: list(range(8))}
for world, rank in [(w, r) for w in (1, 2, 4, 8) for r in ranks_of[w]]:
    plan = StripPlan(c["rows"], c["cols"], c["smax"], c["win"], world, rank)
    g = g_full[plan.g_slice()].contiguous()
    f = torch.empty((plan.f_rows, c["cols"]), dtype=torch.uint8, device="cuda")
    y = torch.empty((plan.core, c["cols"]), dtype=torch.uint8, device="cuda")
    w = torch.zeros(1, dtype=torch.int64, device="cuda")
    be.amf(g, plan, f)
    ta = timed(lambda: be.amf(g, plan, f))
    ts = timed(lambda: be.stats(f, plan, w))
    tg = timed(lambda: be.gain(f, plan, w, y))
    print(f"config {cfg} N={world} rank {rank}: AMF {ta:8.1f} us  stats {ts:7.1f}  gain {tg:7.1f}  "
          f"(x N: {ta * world:8.1f} {ts * world:7.1f} {tg * world:7.1f})")
