"""GPU parity at BASELINE.json's full sizes (configs 2, 3, 4), every pixel checked.

* config 2 (8192^2): the whole hybrid against the oracle (row bands on all host threads).
* config 4 (16384^2, smax 11, S&P 0.5 -- worst-case growth): the GPU's whole AMF output against the
  REFERENCE ITSELF -- adaptive_median_parallel (proj/src/parallel.cpp:27-70, compiled unmodified into
  oracle/_ref) with parts = workers = all host threads (bit-identical to adaptive_median_serial,
  proj/include/denoise/parallel.hpp:27-28) -- then W and every pixel of y against the oracle statistics
  and gain of that f; the GPU hybrid's W and y equal the separate AMF -> statistics -> gain chain.
* config 3 (512 slices of 512^2): the full stack in one batch call, ALL 512 slices against the oracle
  (one slice per host thread), and sampled slices equal to the single-image path.
"""
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2005_05371_b200 import CONFIGS, FilterConfig, capi, denoise

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1


def _phantom(cfg, seed=0):
    c = CONFIGS[cfg]
    return capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], seed)


def test_config2_full_hybrid_vs_oracle(ctx):
    c = CONFIGS[2]
    g = _phantom(2)
    res = denoise.hybrid_denoise(torch.from_numpy(g).cuda(), FilterConfig(smax=c["smax"], wiener_window=c["win"]),
                                 ctx=ctx)
    y = res.image.cpu().numpy()
    ref_y, ref_w = oracle.hybrid_threaded(g, c["smax"], c["win"], THREADS)
    assert res.noise_sum == ref_w
    np.testing.assert_array_equal(y, ref_y)


def test_config4_full_frame_vs_reference(ctx):
    c = CONFIGS[4]
    rows, cols, smax, win = c["rows"], c["cols"], c["smax"], c["win"]
    g = _phantom(4)
    gd = torch.from_numpy(g).cuda()
    f = denoise.adaptive_median_serial(gd, smax, ctx=ctx).cpu().numpy()
    res = denoise.hybrid_denoise(gd, FilterConfig(smax=smax, wiener_window=win), ctx=ctx)
    y = res.image.cpu().numpy()
    if oracle.ref_available():
        ref_f, _ = oracle.ref_amf_parallel(g, smax, parts=THREADS, workers=THREADS)
    else:  # a box without the prebuilt reference library: the oracle restatement (pinned in test_oracle.py)
        ref_f = oracle.amf_threaded(g, smax, THREADS)
    bad = np.argwhere(f != ref_f)
    assert bad.size == 0, f"{len(bad)} AMF pixels differ, first at {bad[:5].tolist()}"
    ref_y, ref_w = oracle.wiener_threaded(f, win, THREADS)
    assert res.noise_sum == ref_w
    np.testing.assert_array_equal(y, ref_y)
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
    refs = oracle.hybrid_many(stack, c["smax"], c["win"], THREADS)
    for s, (ref_y, ref_w) in enumerate(refs):
        assert ws[s] == ref_w, s
        np.testing.assert_array_equal(y[s], ref_y, err_msg=f"slice {s}")
    for s in (1, n // 2 + 1, n - 1):  # the single-image path agrees on more slices
        r = denoise.hybrid_denoise(sd[s], FilterConfig(smax=c["smax"], wiener_window=c["win"]), ctx=ctx)
        assert r.noise_sum == ws[s]
        np.testing.assert_array_equal(r.image.cpu().numpy(), y[s])
