"""GPU: the reference's own Wiener stage -- frequency-domain wiener_filter and
the noise estimates -- against the numpy restatement (oracle/) and the reference's test cases
(proj/tests/test_wiener.cpp:43-192) re-expressed."""
import numpy as np
import pytest
import torch

import oracle
from paper_2005_05371_b200 import capi, denoise

pytestmark = pytest.mark.gpu


def test_zero_variance_returns_the_input(ctx):
    img = np.random.default_rng(30).random((12, 9))
    np.testing.assert_array_equal(denoise.wiener_filter(img, 0.0, clamp=False), img)


def test_negative_variance_rejected_and_all_noise_killed(ctx):
    img = np.random.default_rng(31).random((8, 8))
    with pytest.raises(capi.InvalidArgument, match="nonnegative"):
        denoise.wiener_filter(img, -1e-9)
    tiny = np.zeros((4, 4))
    tiny[1, 2] = 0.01
    assert np.all(np.abs(denoise.wiener_filter(tiny, 1.0, clamp=False)) < 1e-12)


def test_known_cosine_attenuated_by_the_analytic_gain(ctx):
    n = 8
    img = np.tile(np.cos(2 * np.pi * np.arange(n) / n), (n, 1))
    out = denoise.wiener_filter(img, 0.01, clamp=False)
    np.testing.assert_allclose(out, 0.999375 * img, rtol=1e-9, atol=1e-12)


def test_matches_direct_summation_oracle(ctx):
    rng = np.random.default_rng(600)
    for trial in range(12):
        rows, cols = int(rng.integers(2, 9)), int(rng.integers(2, 9))
        img = rng.random((rows, cols))
        sigma2 = 0.002 + 0.004 * (trial % 3)
        fast = denoise.wiener_filter(img, sigma2, clamp=False)
        assert np.max(np.abs(fast - oracle.wiener_direct(img, sigma2))) < 1e-6, trial


def test_never_adds_energy_and_larger_variance_smooths_harder(ctx):
    rng = np.random.default_rng(90)
    img = rng.random((24, 24)) + rng.normal(0.0, 0.1, (24, 24))
    mild = denoise.wiener_filter(img, 0.002, clamp=False)
    strong = denoise.wiener_filter(img, 0.02, clamp=False)
    assert np.sum(mild ** 2) <= np.sum(img ** 2) * (1 + 1e-12)
    assert np.sum(strong ** 2) <= np.sum(mild ** 2) * (1 + 1e-12)
    assert np.all(np.abs(np.fft.fft2(strong)) <= np.abs(np.fft.fft2(mild)) + 1e-9)


def test_clamp_flag_bounds_the_output(ctx):
    img = np.random.default_rng(77).random((6, 6)) * 3.0 - 1.0
    un = denoise.wiener_filter(img, 1e-4, clamp=False)
    cl = denoise.wiener_filter(img, 1e-4, clamp=True)
    assert (un > 1).any() or (un < 0).any()
    np.testing.assert_array_equal(cl, np.clip(un, 0.0, 1.0))


@pytest.mark.parametrize("shape", [(1, 1), (1, 17), (13, 1), (31, 64), (1600, 1600), (257, 1000)])
def test_against_numpy_fft_oracle(ctx, shape):
    img = np.random.default_rng(shape[0] + 3 * shape[1]).random(shape)
    for sigma2, clamp in ((0.003, False), (0.02, True)):
        got = denoise.wiener_filter(img, sigma2, clamp=clamp)
        assert np.max(np.abs(got - oracle.wiener_freq(img, sigma2, clamp))) < 1e-9


def test_device_tensors_and_strided_host_views(ctx):
    base = np.random.default_rng(4).random((40, 50))
    view = base[:, :37]  # pitch 50 elements
    ref = oracle.wiener_freq(np.ascontiguousarray(view), 0.01, True)
    np.testing.assert_allclose(denoise.wiener_filter(view, 0.01), ref, atol=1e-9)
    t = torch.from_numpy(base).cuda()
    out = denoise.wiener_filter(t, 0.01)
    np.testing.assert_allclose(out.cpu().numpy(), oracle.wiener_freq(base, 0.01, True), atol=1e-9)


def test_noise_estimate_reference_mode(ctx):
    a = np.full((8, 8), 0.5)
    b = a.copy()
    b[0, 0] = 0.9
    s2, src = denoise.estimate_noise_variance(a, b)
    assert src == "reference" and abs(s2 - 0.16 / 64) <= 1e-12 * 0.16 / 64
    with pytest.raises(capi.InvalidArgument, match="dimensions do not match"):
        denoise.estimate_noise_variance(a, np.zeros((4, 4)))


def test_noise_estimate_robust_mode(ctx):
    s2, src = denoise.estimate_noise_variance(np.full((32, 32), 0.3))
    assert src == "robust" and s2 == 0.0
    noisy = 0.5 + np.random.default_rng(21).normal(0.0, 0.1, (256, 256))
    s2, _ = denoise.estimate_noise_variance(noisy)
    assert 0.007 < s2 < 0.013
    assert abs(s2 - oracle.noise_robust(noisy)) <= 1e-12 * s2
    odd = np.random.default_rng(5).random((15, 17))  # odd count: the middle element
    assert abs(denoise.estimate_noise_variance(odd)[0] - oracle.noise_robust(odd)) <= 1e-12


def test_contrast_stretch_f64_bit_identical(ctx):
    rng = np.random.default_rng(8)
    for shape in ((1, 1), (5, 5), (300, 517)):
        img = rng.random(shape) * 0.2 + 0.3
        np.testing.assert_array_equal(denoise.contrast_stretch(img), oracle.contrast_stretch_f64(img))
    np.testing.assert_array_equal(denoise.contrast_stretch(np.full((5, 5), 0.42)), np.full((5, 5), 0.42))
    kat = np.array([[0.2, 0.4], [0.6, 0.7]])  # proj/tests/test_pipeline.cpp:29-36
    out = denoise.contrast_stretch(kat)
    assert out[0, 0] == 0.0 and out[1, 1] == 1.0
    np.testing.assert_allclose(out, [[0.0, 0.4], [0.8, 1.0]], rtol=1e-14)


@pytest.mark.parametrize("stretch_after_each", [False, True])
def test_full_reference_pipeline_vs_oracle_chain(ctx, stretch_after_each):
    from paper_2005_05371_b200 import CONFIGS, FilterConfig
    c = CONFIGS[0]
    g = capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)
    res = denoise.hybrid_denoise_reference(g, FilterConfig(smax=c["smax"], parts=4), stretch_after_each=stretch_after_each)
    want, s2 = oracle.hybrid_reference(g, c["smax"], stretch_after_each=stretch_after_each)
    assert abs(res.sigma2 - s2) <= 1e-12 * max(s2, 1e-30)
    assert np.max(np.abs(res.image - want)) < 1e-6  # the reference's own Wiener tolerance
    assert res.image.min() == 0.0 and res.image.max() == 1.0


def test_full_reference_pipeline_reference_mode(ctx):
    from paper_2005_05371_b200 import FilterConfig
    g = capi.make_phantom(200, 260, 8, 12.0, 0.1, 4)
    clean = capi.make_phantom(200, 260, 8, 0.0, 0.0, 4).astype(np.float64) / 255.0
    res = denoise.hybrid_denoise_reference(g, FilterConfig(smax=7), reference=clean)
    want, s2 = oracle.hybrid_reference(g, 7, reference=clean)
    assert abs(res.sigma2 - s2) <= 1e-12 * s2
    assert np.max(np.abs(res.image - want)) < 1e-6
