"""GPU parity at BASELINE.json's full sizes (configs 2, 3, 4), where a whole-image oracle run is too
slow for every case: the GPU computes the FULL workload and the oracle checks it piecewise, with
size-independent properties.

* config 2 (8192^2): the whole hybrid against the oracle (about 15 s of CPU).
* config 4 (16384^2, smax 11, S&P 0.5 -- worst-case growth): the GPU's f against the oracle AMF on
  bands at the top / middle / bottom (the AMF of a row range is defined by the whole source image,
  reference proj/src/adaptive_median.cpp:123-215); W of the GPU's f against the oracle statistics of
  that f; y on the same bands against the oracle gain with that W; and the GPU hybrid's W and y
  equal to the separate AMF -> statistics -> gain chain.
* config 3 (512 slices of 512^2): the full stack in one batch call, 16 sampled slices against the
  oracle, and the whole stack equal to per-slice calls of the single-image path.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2005_05371_b200 import CONFIGS, FilterConfig, capi, denoise

pytestmark = pytest.mark.gpu


def _phantom(cfg, seed=0):
    c = CONFIGS[cfg]
    return capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], seed)


def test_config2_full_hybrid_vs_oracle(ctx):
    c = CONFIGS[2]
    g = _phantom(2)
    res = denoise.hybrid_denoise(torch.from_numpy(g).cuda(), FilterConfig(smax=c["smax"], wiener_window=c["win"]),
                                 ctx=ctx)
    y = res.image.cpu().numpy()
    ref_y, ref_w = oracle.hybrid(g, c["smax"], c["win"])
    assert res.noise_sum == ref_w
    np.testing.assert_array_equal(y, ref_y)


def test_config4_full_size_bands(ctx):
    c = CONFIGS[4]
    rows, cols, smax, win = c["rows"], c["cols"], c["smax"], c["win"]
    g = _phantom(4)
    gd = torch.from_numpy(g).cuda()
    f = denoise.adaptive_median_serial(gd, smax, ctx=ctx).cpu().numpy()
    res = denoise.hybrid_denoise(gd, FilterConfig(smax=smax, wiener_window=win), ctx=ctx)
    y = res.image.cpu().numpy()
    bands = [(0, 192), (rows // 2 - 96, rows // 2 + 96), (rows - 192, rows)]
    for a, b in bands:
        np.testing.assert_array_equal(f[a:b], oracle.amf(g, smax, a, b), err_msg=f"AMF rows [{a},{b})")
    w = oracle.wiener_stats(f, win)
    assert res.noise_sum == w
    for a, b in bands:
        np.testing.assert_array_equal(y[a:b], oracle.wiener_gain(f, win, w, rows * cols, a, b),
                                      err_msg=f"gain rows [{a},{b})")
    # the hybrid call equals the separate AMF -> W1 chain on the GPU everywhere (W and every pixel of y)
    y2, w2 = denoise.wiener_local(torch.from_numpy(f).cuda(), win, ctx=ctx)
    assert w2 == res.noise_sum
    np.testing.assert_array_equal(y2.cpu().numpy(), y)


def test_config3_full_stack(ctx):
    c = CONFIGS[3]
    n = c["slices"]
    stack = np.stack([_phantom(3, s) for s in range(n)])
    sd = torch.from_numpy(stack).cuda()
    y, ws = denoise.hybrid_denoise_batch(sd, c["smax"], c["win"], ctx=ctx)
    y = y.cpu().numpy()
    for s in range(0, n, n // 16):
        ref_y, ref_w = oracle.hybrid(stack[s], c["smax"], c["win"])
        assert ws[s] == ref_w, s
        np.testing.assert_array_equal(y[s], ref_y, err_msg=f"slice {s}")
    for s in (1, n // 2 + 1, n - 1):  # the single-image path agrees on more slices
        r = denoise.hybrid_denoise(sd[s], FilterConfig(smax=c["smax"], wiener_window=c["win"]), ctx=ctx)
        assert r.noise_sum == ws[s]
        np.testing.assert_array_equal(r.image.cpu().numpy(), y[s])
