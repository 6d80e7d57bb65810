"""GPU: randomized parity (hypothesis) of the C-ABI entry points against the oracle over shapes, window
sizes, noise densities, strip counts, row ranges, row pitches and host / device buffers -- every example
bit-exact (AMF, finalized_at, W, y)."""
import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle
from paper_2005_05371_b200 import capi

pytestmark = pytest.mark.gpu
SETTINGS = dict(max_examples=150, deadline=None, derandomize=True,
                suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])
odd = lambda lo, hi: st.integers(lo // 2, hi // 2).map(lambda k: 2 * k + 1)  # noqa: E731


def _img(rows, cols, seed, density):
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 256, size=(rows, cols), dtype=np.uint8) if seed % 3 == 0 else \
        capi.make_phantom(rows, cols, 4, 15.0, 0.0, seed)
    u = rng.random((rows, cols))
    img = base.copy()
    img[u < density / 2] = 0
    img[(u >= density / 2) & (u < density)] = 255
    return img


def _pitched(img, pad, device):
    """img in a buffer whose rows are `pad` bytes longer than the image (strided), on the host or device."""
    rows, cols = img.shape
    buf = np.full((rows, cols + pad), 77, np.uint8)
    buf[:, :cols] = img
    return torch.from_numpy(buf).cuda() if device else buf


def _ptr(b):
    return b.data_ptr() if isinstance(b, torch.Tensor) else b.ctypes.data


def _np(b):
    return b.cpu().numpy() if isinstance(b, torch.Tensor) else b


@settings(**SETTINGS)
@given(rows=st.integers(1, 700), cols=st.integers(1, 900), smax=odd(3, 15), win=odd(1, 9),
       density=st.floats(0.0, 0.9), parts=st.integers(1, 4), pad=st.sampled_from([0, 3, 16, 61]),
       dev_in=st.booleans(), dev_out=st.booleans(), seed=st.integers(0, 10**6))
def test_fuzz_hybrid(ctx, rows, cols, smax, win, density, parts, pad, dev_in, dev_out, seed):
    parts = min(parts, rows)
    g = _img(rows, cols, seed, density)
    gb = _pitched(g, pad, dev_in)
    yb = _pitched(np.zeros_like(g), pad, dev_out)
    stats = capi.HybStats()
    capi.check(capi.lib.hyb_hybrid_u8(ctx.ptr, _ptr(gb), cols + pad, rows, cols, smax, win, parts, _ptr(yb),
                                      cols + pad, capi.ctypes.byref(stats)), ctx.ptr)
    torch.cuda.synchronize()
    ref_y, ref_w = oracle.hybrid(g, smax, win)
    y = _np(yb)
    assert stats.noise_sum == ref_w
    np.testing.assert_array_equal(y[:, :cols], ref_y)
    assert (y[:, cols:] == 77).all()  # the pitch padding is never written


@settings(**SETTINGS)
@given(rows=st.integers(1, 600), cols=st.integers(1, 700), smax=odd(3, 15), density=st.floats(0.0, 0.95),
       lo=st.floats(0.0, 1.0), hi=st.floats(0.0, 1.0), pad=st.sampled_from([0, 5, 32]), dev=st.booleans(),
       seed=st.integers(0, 10**6))
def test_fuzz_amf_rows_and_finalized_at(ctx, rows, cols, smax, density, lo, hi, pad, dev, seed):
    a, b = sorted((int(lo * rows), int(hi * rows)))
    b = max(b, a + 1)
    if b > rows:
        a, b = rows - 1, rows
    g = _img(rows, cols, seed, density)
    gb = _pitched(g, pad, dev)
    fb = _pitched(np.zeros((b - a, cols), np.uint8), pad, dev)
    nb = _pitched(np.zeros((b - a, cols), np.uint8), pad, dev)
    capi.check(capi.lib.hyb_amf_u8(ctx.ptr, _ptr(gb), cols + pad, rows, cols, a, b, smax, _ptr(fb), cols + pad,
                                   _ptr(nb), cols + pad), ctx.ptr)
    torch.cuda.synchronize()
    rf, rn = oracle.amf(g, smax, a, b, finalized_at=True)
    np.testing.assert_array_equal(_np(fb)[:, :cols], rf)
    np.testing.assert_array_equal(_np(nb)[:, :cols], rn)


@settings(**dict(SETTINGS, max_examples=40))
@given(n=st.integers(1, 12), rows=st.integers(1, 300), cols=st.integers(1, 400), smax=odd(3, 13), win=odd(1, 7),
       density=st.floats(0.0, 0.8), dev=st.booleans(), seed=st.integers(0, 10**6))
def test_fuzz_hybrid_batch(ctx, n, rows, cols, smax, win, density, dev, seed):
    stack = np.stack([_img(rows, cols, seed + s, density) for s in range(n)])
    y = np.zeros_like(stack)
    ws = np.zeros(n, np.int64)
    if dev:
        gs, ys = torch.from_numpy(stack).cuda(), torch.from_numpy(y).cuda()
    else:
        gs, ys = stack, y
    capi.check(capi.lib.hyb_hybrid_batch_u8(ctx.ptr, _ptr(gs), cols, rows * cols, n, rows, cols, smax, win,
                                            _ptr(ys), cols, rows * cols,
                                            ws.ctypes.data_as(capi.ctypes.POINTER(capi.ctypes.c_int64))), ctx.ptr)
    torch.cuda.synchronize()
    out = _np(ys)
    for s in range(n):
        ry, rw = oracle.hybrid(stack[s], smax, win)
        assert ws[s] == rw, s
        np.testing.assert_array_equal(out[s], ry, err_msg=f"slice {s}")


@settings(**dict(SETTINGS, max_examples=80))
@given(rows=st.integers(1, 400), cols=st.integers(1, 600), win=odd(1, 15), lo=st.floats(0.0, 1.0),
       hi=st.floats(0.0, 1.0), pad=st.sampled_from([0, 7, 32]), dev=st.booleans(), seed=st.integers(0, 10**6))
def test_fuzz_wiener_row_ranges(ctx, rows, cols, win, lo, hi, pad, dev, seed):
    # W1 statistics and gain on a row range of f (the strip form): W and y against the oracle
    a, b = sorted((int(lo * rows), int(hi * rows)))
    b = max(b, a + 1)
    if b > rows:
        a, b = rows - 1, rows
    f = _img(rows, cols, seed, 0.0)
    fb = _pitched(f, pad, dev)
    w = np.zeros(1, np.int64)
    capi.check(capi.lib.hyb_wiener_stats_u8(ctx.ptr, _ptr(fb), cols + pad, rows, cols, a, b, win, w.ctypes.data),
               ctx.ptr)
    rw = oracle.wiener_stats(f, win, a, b)
    assert int(w[0]) == rw
    yb = _pitched(np.zeros((b - a, cols), np.uint8), pad, dev)
    capi.check(capi.lib.hyb_wiener_gain_u8(ctx.ptr, _ptr(fb), cols + pad, rows, cols, a, b, win, w.ctypes.data,
                                           rows * cols, _ptr(yb), cols + pad), ctx.ptr)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_np(yb)[:, :cols], oracle.wiener_gain(f, win, rw, rows * cols, a, b))


@settings(**dict(SETTINGS, max_examples=60))
@given(rows=st.integers(1, 300), cols=st.integers(1, 300), k=odd(3, 21), density=st.floats(0.0, 0.9),
       dev=st.booleans(), seed=st.integers(0, 10**6))
def test_fuzz_window_stats_and_stretch(ctx, rows, cols, k, density, dev, seed):
    g = _img(rows, cols, seed, density)
    gb = torch.from_numpy(g).cuda() if dev else g
    outs = [torch.empty_like(gb) if dev else np.empty_like(g) for _ in range(3)]
    capi.check(capi.lib.hyb_window_stats_u8(ctx.ptr, _ptr(gb), cols, rows, cols, k, *(_ptr(o) for o in outs), cols),
               ctx.ptr)
    torch.cuda.synchronize()
    for got, want in zip(outs, oracle.window_stats(g, k)):
        np.testing.assert_array_equal(_np(got), want)
    y = torch.empty_like(gb) if dev else np.empty_like(g)
    capi.check(capi.lib.hyb_contrast_stretch_u8(ctx.ptr, _ptr(gb), cols, rows, cols, _ptr(y), cols), ctx.ptr)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_np(y), oracle.contrast_stretch(g))
