"""GPU parity on adversarial inputs: images built to hit the limits of the AMF growth queue and the
W1 integer ranges, on both execution paths (the fused small-image kernel and the separate
k3 -> growth -> statistics -> gain kernels).  Everything is bit-exact against the CPU oracle.

The reference's own tests probe the AMF on ramps, salt on gradients, constants and random images
(proj/tests/test_adaptive_median.cpp:26-130); these add the extremes a GPU implementation has to
survive: every pixel an impulse (level A never passes, so every pixel reaches smax and is never
finalised: the growth queue is full at every level), maximum local variance (0/255 checkerboards:
V = n*S2 - S1^2 at its largest), constant planes, two-level images (many equal values, zmin == zmed),
windows larger than the image, and strided row pitches.
"""
import numpy as np
import pytest

import oracle
from paper_2005_05371_b200 import FilterConfig, capi, denoise

pytestmark = pytest.mark.gpu

# > 888 tiles of 128 x 32 -> the separate-kernel path; <= 888 -> the fused kernel (csrc/small.cu plan_small)
FUSED = (1600, 1600)
SEPARATE = (2048, 2112)


def all_impulse(rows, cols, seed):
    rng = np.random.default_rng(seed)
    return np.where(rng.random((rows, cols)) < 0.5, 0, 255).astype(np.uint8)


def checkerboard(rows, cols, period=1):
    r = (np.arange(rows)[:, None] // period + np.arange(cols)[None, :] // period) & 1
    return (r * 255).astype(np.uint8)


def two_level(rows, cols, seed, density=0.3):
    rng = np.random.default_rng(seed)
    img = rng.integers(0, 2, size=(rows, cols), dtype=np.uint8)
    u = rng.random((rows, cols))
    img[u < density / 2] = 0
    img[(u >= density / 2) & (u < density)] = 255
    return img


def check_hybrid(img, smax, win, parts=1):
    res = denoise.hybrid_denoise(img, FilterConfig(smax=smax, wiener_window=win, parts=parts))
    ref_y, ref_w = oracle.hybrid(img, smax, win)
    assert res.noise_sum == ref_w
    np.testing.assert_array_equal(res.image, ref_y)


@pytest.mark.parametrize("shape", [FUSED, SEPARATE], ids=["fused", "separate"])
@pytest.mark.parametrize("smax,win", [(7, 3), (11, 7)])
def test_hybrid_all_impulse(ctx, shape, smax, win):
    # level A fails everywhere (zmin = 0, zmax = 255, zmed in {0, 255}): every pixel grows to smax
    img = all_impulse(*shape, seed=smax)
    out, fin = denoise.adaptive_median_rows(img, smax, 0, shape[0], finalized_at=True)
    ref_out, ref_fin = oracle.amf(img, smax, finalized_at=True)
    np.testing.assert_array_equal(out, ref_out)
    np.testing.assert_array_equal(fin, ref_fin)
    assert (out == img).all()  # never finalised -> out = g (proj/src/adaptive_median.cpp:134-137)
    check_hybrid(img, smax, win)


@pytest.mark.parametrize("shape", [FUSED, SEPARATE], ids=["fused", "separate"])
@pytest.mark.parametrize("period", [1, 2, 3])
@pytest.mark.parametrize("win", [3, 7])
def test_hybrid_checkerboard_max_variance(ctx, shape, period, win):
    check_hybrid(checkerboard(*shape, period), 7 if win == 3 else 11, win)


@pytest.mark.parametrize("shape", [FUSED, SEPARATE], ids=["fused", "separate"])
@pytest.mark.parametrize("value", [0, 1, 128, 254, 255])
def test_hybrid_constant_planes(ctx, shape, value):
    img = np.full(shape, value, dtype=np.uint8)
    res = denoise.hybrid_denoise(img, FilterConfig(smax=7, wiener_window=3))
    assert res.noise_sum == 0
    assert (res.image == value).all()


@pytest.mark.parametrize("shape", [FUSED, SEPARATE], ids=["fused", "separate"])
@pytest.mark.parametrize("smax,win", [(7, 3), (9, 5)])
def test_hybrid_two_level_images(ctx, shape, smax, win):
    # values {0, 1} plus impulses: zmin == zmed on most windows, so level A fails on flat runs too
    check_hybrid(two_level(*shape, seed=win), smax, win)


@pytest.mark.parametrize("smax", [7, 15])
def test_amf_all_impulse_wide_smax(ctx, smax):
    img = all_impulse(300, 700, seed=smax)
    out, fin = denoise.adaptive_median_rows(img, smax, 0, 300, finalized_at=True)
    ref_out, ref_fin = oracle.amf(img, smax, finalized_at=True)
    np.testing.assert_array_equal(out, ref_out)
    np.testing.assert_array_equal(fin, ref_fin)


@pytest.mark.parametrize("rows,cols", [(1, 17), (5, 5), (17, 1), (3, 200), (200, 3)])
def test_hybrid_window_larger_than_image(ctx, rows, cols):
    img = all_impulse(rows, cols, seed=rows * 31 + cols)
    img[::2, ::3] = 77
    for smax, win in [(15, 7), (11, 5)]:
        check_hybrid(img, smax, win)


@pytest.mark.parametrize("shape", [(513, 777), SEPARATE], ids=["fused", "separate"])
def test_hybrid_strided_rows(ctx, shape):
    # a view into a wider array: row pitch != cols, not a multiple of 16
    rows, cols = shape
    wide = capi.make_phantom(rows, cols + 37, 12, 15.0, 0.2, 5)
    view = wide[:, 11:11 + cols]
    assert view.strides[0] == cols + 37
    res = denoise.hybrid_denoise(view, FilterConfig(smax=7, wiener_window=3))
    ref_y, ref_w = oracle.hybrid(np.ascontiguousarray(view), 7, 3)
    assert res.noise_sum == ref_w
    np.testing.assert_array_equal(res.image, ref_y)


@pytest.mark.parametrize("parts", [2, 4])
def test_hybrid_all_impulse_strips(ctx, parts):
    img = all_impulse(*FUSED, seed=parts)
    check_hybrid(img, 7, 3, parts=parts)


def test_hybrid_batch_adversarial_slices(ctx):
    # one stack mixing the extremes: each slice keeps its own W
    rows, cols = 256, 384
    stack = np.stack([all_impulse(rows, cols, 1), checkerboard(rows, cols), np.full((rows, cols), 9, np.uint8),
                      two_level(rows, cols, 2), capi.make_phantom(rows, cols, 8, 20.0, 0.5, 4)])
    y, ws = denoise.hybrid_denoise_batch(stack, 11, 7)
    for s in range(stack.shape[0]):
        ref_y, ref_w = oracle.hybrid(stack[s], 11, 7)
        assert ws[s] == ref_w, f"slice {s}"
        np.testing.assert_array_equal(y[s], ref_y, err_msg=f"slice {s}")
