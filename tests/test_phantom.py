"""CPU: the BASELINE phantom generator draws from the reference's Rng64 streams exactly
(proj/include/denoise/noise.hpp:24-40, proj/src/noise.cpp:9-62; pins in golden/rng_pins.json)."""
import json
import os

import numpy as np

import oracle
from paper_2005_05371_b200 import capi

PINS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rng_pins.json")))


def lround(x):
    t = np.trunc(x)
    up = ((x - t) >= 0.5).astype(np.float64)
    down = ((t - x) >= 0.5).astype(np.float64)
    return t + np.where(x >= 0, up, -down)


def test_salt_pepper_frozen_draw_502():
    # proj/tests/test_noise.cpp:109-124: 100x100, density 0.05, impulse stream seed 77 -> 502.
    # The generator's impulse stream is seed + 1 (proj/src/noise.cpp:61), so seed 76.
    img = capi.make_phantom(100, 100, 0, 0.0, 0.05, 76)
    assert int(((img == 0) | (img == 255)).sum()) == 502 == PINS["salt_pepper_100x100_d005_seed77"]


def test_impulse_positions_follow_reference_stream():
    rows, cols, d, seed = 20, 30, 0.3, 9
    img = capi.make_phantom(rows, cols, 0, 0.0, d, seed)
    u = oracle.ref_rng(seed + 1, rows * cols).reshape(rows, cols) if oracle.ref_available() else None
    if u is None:
        return
    expect_pepper = u < d / 2
    expect_salt = (u >= d / 2) & (u < d)
    np.testing.assert_array_equal(img == 0, expect_pepper)
    np.testing.assert_array_equal(img == 255, expect_salt)


def test_gaussian_stage_is_exact():
    rows, cols, sigma, seed = 12, 17, 10.0, 7
    img = capi.make_phantom(rows, cols, 0, sigma, 0.0, seed)
    if not oracle.ref_available():
        return
    n = oracle.ref_rng(seed, rows * cols, normal=True).reshape(rows, cols)
    grad = 15.0 * (2.0 * np.arange(cols) / (cols - 1) - 1.0)
    x = (20.0 + grad)[None, :] + sigma * n
    np.testing.assert_array_equal(img, np.clip(lround(x), 0, 255).astype(np.uint8))
    assert list(oracle.ref_rng(7, 16, normal=True)) == PINS["normal_seed7"]


def test_baseline_config_statistics():
    # config 4 flavour: heavy impulses + clipped Gaussian (SURVEY.md 8(d) value distribution)
    img = capi.make_phantom(512, 512, 16, 20.0, 0.5, 0)
    imp = ((img == 0) | (img == 255)).mean()
    assert 0.48 < imp < 0.62
