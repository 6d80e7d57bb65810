"""Per-rank compute time of the multi-GPU strip step (CudaStripBackend) measured on one GPU: for N
strips, the slowest rank's AMF + statistics + gain (CUDA events, device buffers, warm).  With the
halo exchange and the 8-byte all-reduce added, this bounds what `bench.py --gpus N` can reach.
usage: strip_projection.py [config ...]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2005_05371_b200 import CONFIGS, capi  # noqa: E402
from paper_2005_05371_b200.partition import CudaStripBackend, StripPlan  # noqa: E402

ctx = capi.Context(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx.set_stream(s.cuda_stream)
ctx.set_exclusive(True)
be = CudaStripBackend(ctx)
for cfg in [int(a) for a in sys.argv[1:]] or [1, 2, 4]:
    c = CONFIGS[cfg]
    rows, cols = c["rows"], c["cols"]
    g_full = torch.from_numpy(capi.make_phantom(rows, cols, c["ellipses"], c["sigma"], c["density"], 0)).cuda()
    for world in (1, 2, 4, 8):
        worst = 0.0
        for rank in sorted({0, world // 2, world - 1}):
            plan = StripPlan(rows, cols, c["smax"], c["win"], world, rank)
            g = g_full[plan.g_slice()].contiguous()
            f = torch.empty((plan.f_rows, cols), dtype=torch.uint8, device="cuda")
            y = torch.empty((plan.core, cols), dtype=torch.uint8, device="cuda")
            w = torch.zeros(1, dtype=torch.int64, device="cuda")

            def step():
                be.amf(g, plan, f)
                w.zero_()
                be.stats(f, plan, w)
                be.gain(f, plan, w, y)
            for _ in range(5):
                step()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                step()
            e1.record()
            torch.cuda.synchronize()
            worst = max(worst, e0.elapsed_time(e1) / 20 * 1e3)
        mpix = rows * cols / worst
        print(f"config {cfg} N={world}: slowest strip compute {worst:8.1f} us -> {mpix:9.0f} MPix/s aggregate "
              f"(compute only, no exchange / all-reduce)")
