"""Multi-device context (hyb_create_multi) through the C ABI: one strip per listed device, NVLink
exchange of the partial noise sums, bit-identical to one device.  The pool has one GPU per box, so the
strips run as several contexts on device 0 (ids repeat: separate streams, the same code path --
cross-device events, the W reduction kernel reading every strip's partial, direct or staged output);
on a box with >= 2 GPUs the same tests also run across real devices."""
import numpy as np
import pytest
import torch

import oracle
from paper_2005_05371_b200 import CONFIGS, FilterConfig, capi, denoise

pytestmark = pytest.mark.gpu


def _img(rows, cols, seed, density=0.3):
    return capi.make_phantom(rows, cols, 16, 12.0, density, seed)


def _device_sets():
    sets = [[0, 0], [0, 0, 0], [0] * 8]
    n = torch.cuda.device_count()
    if n >= 2:
        sets += [list(range(n)), [i % n for i in range(8)]]
    return sets


@pytest.mark.parametrize("devices", _device_sets())
@pytest.mark.parametrize("shape,smax,win", [((2053, 1500), 9, 5), ((611, 997), 11, 7), ((64, 300), 7, 3)])
def test_multi_hybrid_device_buffers_bit_identical(devices, shape, smax, win):
    g = _img(*shape, seed=shape[0] + len(devices))
    ref_y, ref_w = oracle.hybrid_threaded(g, smax, win)
    mc = capi.Context(devices=devices)
    assert mc.devices() == devices
    gd = torch.from_numpy(g).cuda()
    res = denoise.hybrid_denoise(gd, FilterConfig(smax=smax, wiener_window=win), ctx=mc)
    assert res.noise_sum == ref_w
    np.testing.assert_array_equal(res.image.cpu().numpy(), ref_y)
    mc.close()


@pytest.mark.parametrize("devices", _device_sets()[:2])
def test_multi_hybrid_host_buffers_and_strided(devices):
    g = _img(1777, 1203, 7)
    ref_y, ref_w = oracle.hybrid_threaded(g, 9, 5)
    mc = capi.Context(devices=devices)
    res = denoise.hybrid_denoise(g, FilterConfig(smax=9, wiener_window=5), ctx=mc)  # numpy in, numpy out
    assert res.noise_sum == ref_w
    np.testing.assert_array_equal(res.image, ref_y)
    # strided host rows (pitch > cols)
    big = np.zeros((1777, 1300), np.uint8)
    big[:, :1203] = g
    view = big[:, :1203]
    res2 = denoise.hybrid_denoise(view, FilterConfig(smax=9, wiener_window=5), ctx=mc)
    np.testing.assert_array_equal(res2.image, ref_y)
    mc.close()


def test_multi_config4_eight_strips_equal_single_device(ctx):
    c = CONFIGS[4]
    g = capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)
    gd = torch.from_numpy(g).cuda()
    cfg = FilterConfig(smax=c["smax"], wiener_window=c["win"])
    one = denoise.hybrid_denoise(gd, cfg, ctx=ctx)
    mc = capi.Context(devices=[0] * 8)
    many = denoise.hybrid_denoise(gd, cfg, ctx=mc)
    assert many.noise_sum == one.noise_sum
    assert torch.equal(many.image, one.image)
    mc.close()


@pytest.mark.parametrize("devices", _device_sets()[:2])
def test_multi_batch_shards_slices(devices):
    stack = np.stack([_img(256, 320, s, 0.1) for s in range(37)])
    refs = oracle.hybrid_many(stack, 7, 3)
    mc = capi.Context(devices=devices)
    for src in (torch.from_numpy(stack).cuda(), stack):
        y, ws = denoise.hybrid_denoise_batch(src, 7, 3, ctx=mc)
        y = y.cpu().numpy() if hasattr(y, "cpu") else y
        for s, (ry, rw) in enumerate(refs):
            assert ws[s] == rw, s
            np.testing.assert_array_equal(y[s], ry, err_msg=f"slice {s}")
    mc.close()


def test_multi_errors_keep_reference_text():
    mc = capi.Context(devices=[0, 0, 0])
    g = torch.zeros((2, 50), dtype=torch.uint8, device="cuda")
    with pytest.raises(capi.InvalidArgument, match="exceeds image rows"):
        denoise.hybrid_denoise(g, FilterConfig(smax=7, wiener_window=3), ctx=mc)
    with pytest.raises(capi.InvalidArgument, match="odd integer > 1"):
        denoise.hybrid_denoise(torch.zeros((64, 64), dtype=torch.uint8, device="cuda"),
                               FilterConfig(smax=4, wiener_window=3), ctx=mc)
    mc.close()


def test_config_gpus_and_device_ids_route_to_multi_context():
    g = _img(900, 700, 11)
    ref_y, ref_w = oracle.hybrid_threaded(g, 9, 5)
    res = denoise.hybrid_denoise(g, FilterConfig(smax=9, wiener_window=5, device_ids=(0, 0, 0)))
    assert res.noise_sum == ref_w
    np.testing.assert_array_equal(res.image, ref_y)
    if torch.cuda.device_count() >= 2:
        res = denoise.hybrid_denoise(g, FilterConfig(smax=9, wiener_window=5, gpus=torch.cuda.device_count()))
        np.testing.assert_array_equal(res.image, ref_y)


def test_estimate_mode_reference_and_stretches():
    """The reference's hybrid_denoise options (proj/include/denoise/pipeline.hpp:25-27): estimate_mode
    REFERENCE (sigma2 = mean squared difference to the reference image), stretch_after_each, and the
    closing contrast stretch -- each checked against the oracle chain."""
    rows, cols = 140, 170
    g = _img(rows, cols, 12, 0.2)
    f = oracle.amf(g, 7)
    clean = np.tile((20.0 + 0.5 * np.arange(cols)) / 255.0, (rows, 1))
    with pytest.raises(capi.InvalidArgument, match="reference mode requires a reference image"):
        denoise.hybrid_denoise(g, FilterConfig(smax=7, estimate_mode=denoise.EstimateMode.REFERENCE))
    with pytest.raises(capi.InvalidArgument, match="dimensions do not match"):
        denoise.hybrid_denoise(g, FilterConfig(smax=7), reference=clean[:10])
    for src in (g, torch.from_numpy(g).cuda()):
        res = denoise.hybrid_denoise(src, FilterConfig(smax=7, wiener_window=3,
                                                       estimate_mode=denoise.EstimateMode.REFERENCE), reference=clean)
        sigma2 = float(np.mean((f / 255.0 - clean) ** 2))
        assert abs(res.sigma2 - sigma2) <= 1e-12
        pn = rows * cols * 64
        w = int(np.floor(sigma2 * 255.0 * 255.0 * 81 * pn + 0.5))
        y = res.image.cpu().numpy() if hasattr(res.image, "cpu") else res.image
        np.testing.assert_array_equal(y, oracle.wiener_gain(f, 3, w, pn))
    fs = oracle.contrast_stretch(f)
    ys, ws = oracle.wiener(fs, 3)
    res = denoise.hybrid_denoise(g, FilterConfig(smax=7, wiener_window=3, final_stretch=True), stretch_after_each=True)
    assert res.noise_sum == ws
    np.testing.assert_array_equal(res.image, oracle.contrast_stretch(ys))


@pytest.mark.parametrize("devices", [None] + _device_sets()[:2])
@pytest.mark.parametrize("shape,smax,win,parts", [((2053, 1500), 9, 5, 1), ((611, 997), 11, 7, 1),
                                                  ((300, 400), 7, 9, 1), ((1100, 900), 7, 3, 3),
                                                  ((64, 300), 5, 3, 1)])
def test_hybrid_stretch_fused_range(ctx, devices, shape, smax, win, parts):
    # stages 1-3 (reference proj/src/pipeline.cpp:23-57): the contrast stretch's min / max folded into the
    # W1 gain (separate-kernel path; the generic gain for win 9 and the fused small-image kernel take a
    # separate min / max pass), and across strips the per-device ranges combined over NVLink before each
    # strip maps its own rows (multi-device contexts) -- all equal to the oracle's stretch of the oracle
    g = _img(*shape, seed=shape[1] + smax)
    g[:3, :5] = 0  # the full range present, and not: both map branches exercised across cases
    if shape[0] == 64:
        g[g > 200] = 200
    ref_y, ref_w = oracle.hybrid_threaded(g, smax, win)
    want = oracle.contrast_stretch(ref_y)
    c = ctx if devices is None else capi.Context(devices=devices)
    cfg = FilterConfig(smax=smax, wiener_window=win, parts=parts if devices is None else 1)
    res = denoise.hybrid_denoise_stretched(torch.from_numpy(g).cuda(), cfg, ctx=c)
    assert res.noise_sum == ref_w
    np.testing.assert_array_equal(res.image.cpu().numpy(), want)
    res = denoise.hybrid_denoise_stretched(g, cfg, ctx=c)  # host buffers
    np.testing.assert_array_equal(res.image, want)
    if devices is not None:
        c.close()
