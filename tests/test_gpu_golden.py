"""GPU: the CUDA path (through the C ABI) against the REFERENCE's own outputs (tests/golden,
generated from the reference compiled from /root/reference; no reference code is needed here)."""
import json
import os

import numpy as np
import pytest

from paper_2005_05371_b200 import FilterConfig, denoise

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "amf_reference.npz"))


def test_amf_all_reference_fixtures(ctx, gold):
    names = sorted({k.split("/")[0] for k in gold.files})
    n = 0
    for name in names:
        img = gold[f"{name}/input"]
        for key in gold.files:
            if key.startswith(name + "/out_s"):
                smax = int(key.split("_s")[-1])
                out, fin = denoise.adaptive_median_rows(img, smax, 0, img.shape[0], finalized_at=True)
                np.testing.assert_array_equal(out, gold[key], err_msg=f"{name} smax={smax}")
                np.testing.assert_array_equal(fin, gold[f"{name}/fin_s{smax}"], err_msg=f"{name} smax={smax}")
                n += 1
    assert n > 500


def test_amf_parallel_grid_against_reference(ctx, gold):
    # acceptance criterion 1 (proj/tests/acceptance.cpp:50-80): every parts is bit-identical to serial
    for t in range(0, 20, 3):
        img = gold[f"exact20_{t:02d}/input"]
        for smax in (3, 7, 11):
            ref = gold[f"exact20_{t:02d}/out_s{smax}"]
            for parts in (1, 2, 4, 8):
                out = denoise.adaptive_median_parallel(img, FilterConfig(smax=smax, parts=parts, workers=parts))
                np.testing.assert_array_equal(out, ref, err_msg=f"{t} smax={smax} parts={parts}")


def test_amf_halo_free_split_matches_reference(ctx, gold):
    # proj/tests/test_parallel.cpp:86-103: use_halo = false reproduces the literal halo-free split
    img = gold["par_40x40_s6/input"]
    out = denoise.adaptive_median_parallel(img, FilterConfig(smax=11, parts=4, workers=2, use_halo=False))
    np.testing.assert_array_equal(out, gold["par_40x40_s6/nohalo_p4_s11"])
    assert (out != gold["par_40x40_s6/out_s11"]).any()


def test_wiener_kats(ctx):
    for k in json.load(open(os.path.join(GOLD, "wiener_kat.json"))):
        f = np.array(k["f"], np.uint8)
        y, w = denoise.wiener_local(f, k["win"])
        assert w == k["W"], k["name"]
        np.testing.assert_array_equal(y, np.array(k["y"], np.uint8), err_msg=k["name"])
