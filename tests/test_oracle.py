"""CPU: the C oracle against the reference's golden vectors (tests/golden, generated from the
reference itself by make_golden.py) and against the reference live where oracle/_ref is built."""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def amf_gold():
    return np.load(os.path.join(GOLD, "amf_reference.npz"))


def cases(gold):
    names = sorted({k.split("/")[0] for k in gold.files})
    for name in names:
        img = gold[f"{name}/input"]
        for key in gold.files:
            if key.startswith(name + "/out_s"):
                smax = int(key.split("_s")[-1])
                yield name, img, smax, gold[key], gold[f"{name}/fin_s{smax}"]


def test_oracle_amf_matches_reference_golden(amf_gold):
    n = 0
    for name, img, smax, out, fin in cases(amf_gold):
        o, f = oracle.amf(img, smax, finalized_at=True)
        np.testing.assert_array_equal(o, out, err_msg=f"{name} smax={smax}")
        np.testing.assert_array_equal(f, fin, err_msg=f"{name} smax={smax}")
        n += 1
    assert n > 500


def test_reference_kats(amf_gold):
    # proj/tests/test_adaptive_median.cpp:67-78: the salt impulse becomes the window median (0.5 -> 5)
    assert amf_gold["kat_gradient_salt/out_s3"][2, 2] == 5
    np.testing.assert_array_equal(amf_gold["kat_constant/out_s11"], amf_gold["kat_constant/input"])


def test_oracle_finalized_at_invariants(amf_gold):
    # proj/tests/test_adaptive_median.cpp:108-130
    img = amf_gold["fin_20x20_70/input"]
    o5, f5 = oracle.amf(img, 5, finalized_at=True)
    o11, f11 = oracle.amf(img, 11, finalized_at=True)
    m = f5 != 0
    assert set(np.unique(f5)) <= {0, 3, 5}
    np.testing.assert_array_equal(f11[m], f5[m])
    np.testing.assert_array_equal(o11[m], o5[m])
    np.testing.assert_array_equal(o11[f11 == 0], img[f11 == 0])


def test_oracle_output_in_input_multiset(amf_gold):
    img = amf_gold["par_30x26_700/input"]
    out = oracle.amf(img, 7)
    assert np.isin(out, img).all()


def test_oracle_row_ranges_compose():
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, (41, 37), dtype=np.uint8)
    img[rng.random(img.shape) < 0.3] = 255
    full = oracle.amf(img, 9)
    parts = [oracle.amf(img, 9, a, b) for a, b in [(0, 7), (7, 30), (30, 41)]]
    np.testing.assert_array_equal(np.vstack(parts), full)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(6))
def test_oracle_matches_reference_live(seed):
    rng = np.random.default_rng(seed)
    rows, cols = int(rng.integers(1, 70)), int(rng.integers(1, 90))
    img = oracle.ref_random_image(rows, cols, 100 + seed, 0.35, 200 + seed)
    for smax in (3, 5, 9, 13, 21):
        o, f = oracle.amf(img, smax, finalized_at=True)
        r, rf = oracle.ref_amf_rows(img, smax, finalized_at=True)
        np.testing.assert_array_equal(o, r)
        np.testing.assert_array_equal(f, rf)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_reference_parallel_is_partition_invariant_on_grid():
    img = oracle.ref_noisy_phantom(64, 64, 3)
    serial = oracle.ref_amf_rows(img, 11)
    for parts in (2, 3, 4, 8):
        out, _ = oracle.ref_amf_parallel(img, 11, parts, 4)
        np.testing.assert_array_equal(out, serial)


def test_validate_smax():
    for good in (3, 11, 255):
        assert oracle.lib().hyb_oracle_validate_smax(good) == 0
    for bad in (4, 1, 0, -3):
        assert oracle.lib().hyb_oracle_validate_smax(bad) != 0


# ---------------------------------------------------------------- W1

def test_oracle_wiener_kats():
    with open(os.path.join(GOLD, "wiener_kat.json")) as fh:
        kats = json.load(fh)
    for k in kats:
        f = np.array(k["f"], np.uint8)
        y, w = oracle.wiener(f, k["win"])
        assert w == k["W"], k["name"]
        np.testing.assert_array_equal(y, np.array(k["y"], np.uint8), err_msg=k["name"])


def test_oracle_wiener_constant_is_identity():
    f = np.full((12, 9), 77, np.uint8)
    y, w = oracle.wiener(f, 5)
    assert w == 0
    np.testing.assert_array_equal(y, f)


def test_oracle_wiener_output_within_window_range():
    rng = np.random.default_rng(7)
    f = rng.integers(0, 256, (30, 40), dtype=np.uint8)
    for win in (3, 5, 7):
        y, _ = oracle.wiener(f, win)
        r = win // 2
        pad = np.pad(f, r, mode="edge")
        win_min = np.min([pad[i:i + 30, j:j + 40] for i in range(win) for j in range(win)], axis=0)
        win_max = np.max([pad[i:i + 30, j:j + 40] for i in range(win) for j in range(win)], axis=0)
        assert (y >= win_min).all() and (y <= win_max).all()


def test_oracle_wiener_noise_sum_is_partition_invariant():
    rng = np.random.default_rng(11)
    f = rng.integers(0, 256, (57, 33), dtype=np.uint8)
    for win in (3, 7):
        whole = oracle.wiener_stats(f, win)
        cuts = [0, 5, 19, 20, 44, 57]
        assert sum(oracle.wiener_stats(f, win, a, b) for a, b in zip(cuts, cuts[1:])) == whole


# W1 pinned to a published third-party implementation: scipy.signal.wiener (scipy 1.x, the MATLAB
# wiener2 estimator: local mean / variance over an N x N box, noise = the mean local variance, output
# lMean where lVar < noise, else lMean + (1 - noise / lVar) (im - lMean)).  Edge replication is supplied
# by padding the image (scipy pads with zeros, which the crop removes); the noise is passed as the
# oracle's exact nu = W / (n^2 P).  scipy computes in float64; the result is rounded half up.
def _scipy_w1(f, win, nu):
    from scipy.signal import wiener as sp_wiener
    r = win // 2
    pad = np.pad(f.astype(np.float64), r, mode="edge")
    with np.errstate(divide="ignore", invalid="ignore"):
        out = sp_wiener(pad, (win, win), noise=nu)
    out = out[r:r + f.shape[0], r:r + f.shape[1]] if r else out
    return np.clip(np.floor(out + 0.5), 0, 255).astype(np.uint8)


@pytest.mark.parametrize("win", [3, 5, 7])
@pytest.mark.parametrize("seed,shape,sp", [(0, (97, 131), 0.0), (1, (64, 200), 0.1), (2, (150, 77), 0.3)])
def test_oracle_wiener_matches_scipy_signal_wiener(win, seed, shape, sp):
    pytest.importorskip("scipy")
    from numpy.lib.stride_tricks import sliding_window_view
    rng = np.random.default_rng(seed)
    base = np.clip(rng.normal(120, 40, shape), 0, 255)
    u = rng.random(shape)
    base[u < sp / 2] = 0
    base[(u >= sp / 2) & (u < sp)] = 255
    f = np.floor(base + 0.5).astype(np.uint8)
    y, w = oracle.wiener(f, win)
    n, P = win * win, f.size
    nu = w / (n * n * P)
    # nu equals numpy's mean local variance (edge-replicated windows)
    r = win // 2
    wins = sliding_window_view(np.pad(f.astype(np.float64), r, mode="edge"), (win, win))
    lvar = wins.var(axis=(2, 3))
    assert abs(nu - lvar.mean()) <= 1e-9 * max(1.0, nu)
    ys = _scipy_w1(f, win, nu)
    d = np.abs(y.astype(np.int16) - ys.astype(np.int16))
    # north_star tolerance (<= 1 LSB, >= 99.99 % exact); the exact-rational oracle agrees bit for bit
    assert d.max() <= 1 and (d == 0).mean() >= 0.9999
    np.testing.assert_array_equal(y, ys)


# ---------------------------------------------------------------- contrast_stretch

def _stretch_ref_double(img):
    """The reference's double formula (proj/src/pipeline.cpp:10-21) on k/255 values."""
    p = img.astype(np.float64) / 255.0
    lo, hi = p.min(), p.max()
    if hi == lo:
        return p
    return (p - lo) / (hi - lo)


def test_contrast_stretch_kat_range_onto_0_1():
    # proj/tests/test_pipeline.cpp:29-36 on the k/255 grid: {0.2, 0.4, 0.6, 0.7}
    img = np.array([[51, 102], [153, 179]], np.uint8)
    out = oracle.contrast_stretch(img)
    assert out[0, 0] == 0 and out[1, 1] == 255
    np.testing.assert_array_equal(out, np.floor(_stretch_ref_double(img) * 255 + 0.5).astype(np.uint8))


def test_contrast_stretch_constants_and_full_range_unchanged():
    # proj/tests/test_pipeline.cpp:38-43
    flat = np.full((5, 5), 107, np.uint8)
    np.testing.assert_array_equal(oracle.contrast_stretch(flat), flat)
    full = np.array([[0, 64, 255]], np.uint8)
    np.testing.assert_array_equal(oracle.contrast_stretch(full), full)


def test_contrast_stretch_endpoints_order_and_rounding():
    # proj/tests/test_pipeline.cpp:45-57: both endpoints, order preserved; plus: the uint8 value is the
    # reference's double result scaled by 255 and rounded to nearest (ties: exact rational, half up)
    rng = np.random.default_rng(321)
    for lo, hi in ((76, 128), (0, 17), (200, 255), (3, 250)):
        img = rng.integers(lo, hi + 1, size=(13, 11), dtype=np.uint8)
        img[0, 0], img[-1, -1] = lo, hi
        out = oracle.contrast_stretch(img)
        assert out.min() == 0 and out.max() == 255
        flat_in, flat_out = img.ravel().astype(int), out.ravel().astype(int)
        order = np.argsort(flat_in, kind="stable")
        assert np.all(np.diff(flat_out[order]) >= 0)
        ref = _stretch_ref_double(img) * 255.0
        assert np.max(np.abs(out - ref)) <= 0.5 + 1e-9
        exact = (510 * (img.astype(int) - lo) + (hi - lo)) // (2 * (hi - lo))
        np.testing.assert_array_equal(out, exact)


# ---------------------------------------------------------------- window_stats

def ws_cases():
    gold = np.load(os.path.join(GOLD, "window_stats_reference.npz"))
    for key in gold.files:
        if "/k" in key:
            name, k = key.split("/k")
            yield name, gold[f"{name}/input"], int(k), gold[key]


def test_oracle_window_stats_matches_reference_golden():
    n = 0
    for name, img, k, planes in ws_cases():
        got = np.stack(oracle.window_stats(img, k))
        np.testing.assert_array_equal(got, planes, err_msg=f"{name} k={k}")
        n += 1
    assert n >= 20


def test_oracle_window_stats_kats():
    # proj/tests/test_adaptive_median.cpp:26-48 (rank-compressed ramp), invalid sizes
    zmin, zmed, zmax = oracle.window_stats(np.arange(1, 10, dtype=np.uint8).reshape(3, 3), 3)
    assert (zmin[1, 1], zmed[1, 1], zmax[1, 1]) == (1, 5, 9)
    assert (zmin[0, 0], zmed[0, 0], zmax[0, 0]) == (1, 2, 5)
    for k in (4, 1):
        with pytest.raises(ValueError):
            oracle.window_stats(np.zeros((6, 5), np.uint8), k)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("k", [3, 5, 9, 13])
def test_oracle_window_stats_live_vs_reference(k):
    rng = np.random.default_rng(k)
    img = rng.integers(0, 256, size=(37, 45), dtype=np.uint8)
    img[rng.random(img.shape) < 0.2] = 255
    for a, b in zip(oracle.window_stats(img, k), oracle.ref_window_stats(img, k)):
        np.testing.assert_array_equal(a, b)
