"""GPU: the multi-GPU strip step's per-rank compute (CudaStripBackend, the product backend of
partition.py) on one GPU, ranks run one after another in this process.  The halo exchange is
replaced by slicing the image (the exchange itself is tested over gloo in test_partition_gloo.py)
and the all-reduce by a sum of the ranks' noise sums.  The stitched strips must equal the
single-image hybrid bit for bit -- what `bench.py --gpus N` computes on N GPUs."""
import numpy as np
import pytest
import torch

import oracle
from paper_2005_05371_b200 import CONFIGS, FilterConfig, capi, denoise
from paper_2005_05371_b200.partition import CudaStripBackend, StripPlan

pytestmark = pytest.mark.gpu


def _strip_hybrid(ctx, img, smax, win, world):
    rows, cols = img.shape
    h = torch.cuda.current_stream().cuda_stream
    ctx.set_stream(h if h else 1)  # the backend's kernels on torch's stream (as bench.py does)
    backend = CudaStripBackend(ctx)
    gd = torch.from_numpy(img).cuda()
    plans, fs, ws = [], [], []
    for rank in range(world):
        plan = StripPlan(rows, cols, smax, win, world, rank)
        g = gd[plan.g_slice()].contiguous()  # own core rows + the halo rows the exchange delivers
        f = torch.empty((plan.f_rows, cols), dtype=torch.uint8, device="cuda")
        w = torch.zeros(1, dtype=torch.int64, device="cuda")
        backend.amf(g, plan, f)
        backend.stats(f, plan, w)
        plans.append(plan)
        fs.append(f)
        ws.append(w)
    w_all = torch.stack(ws).sum(0)  # the all-reduce
    y = torch.empty_like(gd)
    for plan, f in zip(plans, fs):
        backend.gain(f, plan, w_all, y[plan.core_slice()])
    return y.cpu().numpy(), int(w_all.item())


@pytest.mark.parametrize("world", [2, 4, 8])
def test_strip_backend_config1_matches_single_gpu(ctx, world):
    c = CONFIGS[1]
    img = capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)
    ref = denoise.hybrid_denoise(torch.from_numpy(img).cuda(), FilterConfig(smax=c["smax"], wiener_window=c["win"]),
                                 ctx=ctx)
    y, w = _strip_hybrid(ctx, img, c["smax"], c["win"], world)
    assert w == ref.noise_sum
    np.testing.assert_array_equal(y, ref.image.cpu().numpy())


@pytest.mark.parametrize("world", [3, 8])
def test_strip_backend_config4_statistics_vs_oracle(ctx, world):
    # config-4 statistics (sigma 20, S&P 0.5, smax 11, Wiener 7x7) on a 1024 x 768 phantom
    img = capi.make_phantom(1024, 768, 16, 20.0, 0.5, 1)
    ref_y, ref_w = oracle.hybrid(img, 11, 7)
    y, w = _strip_hybrid(ctx, img, 11, 7, world)
    assert w == ref_w
    np.testing.assert_array_equal(y, ref_y)
