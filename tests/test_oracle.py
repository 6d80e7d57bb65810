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
