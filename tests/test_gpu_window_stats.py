"""GPU: window_stats (reference proj/src/adaptive_median.cpp:96-119) through the
C ABI (hyb_window_stats_u8) against the C oracle, bit-exact; the reference's own cases
(proj/tests/test_adaptive_median.cpp:26-59) re-expressed on uint8."""
import numpy as np
import pytest
import torch

import oracle
from paper_2005_05371_b200 import capi, denoise

pytestmark = pytest.mark.gpu


def test_window_stats_ramp_kat(ctx):
    # proj/tests/test_adaptive_median.cpp:26-38, rank-compressed 0.1..0.9 -> 1..9
    img = np.arange(1, 10, dtype=np.uint8).reshape(3, 3)
    ws = denoise.window_stats(img, 3)
    assert ws.k == 3
    assert (ws.zmin[1, 1], ws.zmed[1, 1], ws.zmax[1, 1]) == (1, 5, 9)
    # corner multiset {1 x4, 2 x2, 4 x2, 5}: the fifth element is 2
    assert (ws.zmin[0, 0], ws.zmed[0, 0], ws.zmax[0, 0]) == (1, 2, 5)


def test_window_stats_constant_and_invalid(ctx):
    # :40-48
    flat = np.full((6, 5), 64, np.uint8)
    ws = denoise.window_stats(flat, 5)
    for p in (ws.zmin, ws.zmed, ws.zmax):
        np.testing.assert_array_equal(p, flat)
    for k in (4, 1, 0, -3):
        with pytest.raises(capi.InvalidArgument, match="odd integer >= 3"):
            denoise.window_stats(flat, k)
    # the C ABI itself rejects it with the reference's text
    out = np.empty_like(flat)
    st = capi.lib.hyb_window_stats_u8(ctx.ptr, flat.ctypes.data, 5, 6, 5, 4, out.ctypes.data, None, None, 5)
    assert st == capi.HYB_EINVAL and b"got 4" in capi.lib.hyb_last_error(ctx.ptr)


@pytest.mark.parametrize("shape,k", [((21, 17), 3), ((21, 17), 5), ((21, 17), 7), ((1, 1), 3), ((1, 300), 5),
                                     ((300, 1), 7), ((97, 131), 9), ((97, 131), 11), ((33, 70), 15),
                                     ((40, 50), 101), ((40, 50), 201), ((515, 1030), 5)])
def test_window_stats_vs_oracle(ctx, shape, k):
    # :50-59 ordering invariant, and every plane bit-exact vs the oracle (incl. the global-memory path,
    # k > 193, and windows much larger than the image)
    rng = np.random.default_rng(shape[0] * 31 + shape[1] + k)
    img = rng.integers(0, 256, size=shape, dtype=np.uint8)
    u = rng.random(shape)
    img[u < 0.1] = 0
    img[(u >= 0.1) & (u < 0.2)] = 255
    ws = denoise.window_stats(img, k)
    ref = oracle.window_stats(img, k)
    assert (ws.zmin <= ws.zmed).all() and (ws.zmed <= ws.zmax).all()
    for got, want in zip((ws.zmin, ws.zmed, ws.zmax), ref):
        np.testing.assert_array_equal(got, want)


def test_window_stats_device_strided_and_nullable(ctx):
    rng = np.random.default_rng(7)
    base = rng.integers(0, 256, size=(80, 160), dtype=np.uint8)
    view = base[5:70, 9:140]  # strided host view
    ref = oracle.window_stats(np.ascontiguousarray(view), 7)
    ws = denoise.window_stats(view, 7)
    for got, want in zip((ws.zmin, ws.zmed, ws.zmax), ref):
        np.testing.assert_array_equal(got, want)
    # device input and outputs, only the median plane requested, outputs at a padded pitch
    g = torch.from_numpy(np.ascontiguousarray(view)).cuda()
    rows, cols = g.shape
    med = torch.full((rows, 160), 77, dtype=torch.uint8, device="cuda")
    capi.check(capi.lib.hyb_window_stats_u8(ctx.ptr, g.data_ptr(), cols, rows, cols, 7, None, med.data_ptr(), None,
                                            160), ctx.ptr)
    torch.cuda.synchronize()
    m = med.cpu().numpy()
    np.testing.assert_array_equal(m[:, :cols], ref[1])
    assert (m[:, cols:] == 77).all()  # pitch padding untouched
    # mixed: device input, host min plane + device max plane
    hmin = np.empty((rows, cols), np.uint8)
    dmax = torch.empty((rows, cols), dtype=torch.uint8, device="cuda")
    capi.check(capi.lib.hyb_window_stats_u8(ctx.ptr, g.data_ptr(), cols, rows, cols, 7, hmin.ctypes.data, None,
                                            dmax.data_ptr(), cols), ctx.ptr)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(hmin, ref[0])
    np.testing.assert_array_equal(dmax.cpu().numpy(), ref[2])


def test_window_stats_vs_reference_golden(ctx):
    # planes generated from the reference itself (tests/golden/make_golden.py)
    import os
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "window_stats_reference.npz"))
    n = 0
    for key in gold.files:
        if "/k" not in key:
            continue
        name, k = key.split("/k")
        ws = denoise.window_stats(gold[f"{name}/input"], int(k))
        np.testing.assert_array_equal(np.stack([ws.zmin, ws.zmed, ws.zmax]), gold[key], err_msg=key)
        n += 1
    assert n >= 20
