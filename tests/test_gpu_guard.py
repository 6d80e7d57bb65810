"""Out-of-bounds write checks without compute-sanitizer (closed on the GPU pool): every entry point
writes into a strided view of a larger device buffer filled with a canary byte, and the test checks
that (1) the view holds the oracle's result and (2) every byte outside the view -- guard rows above and
below, the pitch padding left and right of each row, the gaps between stack slices -- still holds the
canary.  The same is done for the inputs, which must come back unmodified.
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle
from paper_2005_05371_b200 import capi

pytestmark = pytest.mark.gpu

CANARY = 0xA5
LPAD, RPAD, GUARD = 16, 45, 3


def guarded(rows, cols, dev="cuda", init=None):
    """(full buffer, view): view = rows x cols at (GUARD, LPAD) of a canary-filled buffer on the device,
    in pinned host memory (dev="pinned") or in pageable host memory (dev="cpu")."""
    full = torch.full((rows + 2 * GUARD, LPAD + cols + RPAD), CANARY, dtype=torch.uint8,
                      device="cpu" if dev == "pinned" else dev)
    if dev == "pinned":
        full = full.pin_memory()
    view = full[GUARD:GUARD + rows, LPAD:LPAD + cols]
    if init is not None:
        view.copy_(torch.from_numpy(init))
    return full, view


def outside(full, rows, cols):
    m = torch.ones_like(full, dtype=torch.bool)
    m[GUARD:GUARD + rows, LPAD:LPAD + cols] = False
    return full[m]


def assert_guards(full, rows, cols, what):
    o = outside(full, rows, cols)
    bad = int((o != CANARY).sum())
    assert bad == 0, f"{what}: {bad} bytes outside the view were written"


def run(st, ctx, what):
    torch.cuda.synchronize()
    capi.check(st, ctx.ptr)
    torch.cuda.synchronize()


@pytest.mark.parametrize("rows,cols,smax,win", [(300, 333, 7, 3), (1600, 1600, 11, 7), (2048, 2112, 9, 5),
                                                 (5, 3, 15, 7), (1, 200, 7, 3)])
@pytest.mark.parametrize("parts", [1, 2])
@pytest.mark.parametrize("mem", ["cuda", "pinned", "cpu"])
def test_hybrid_writes_stay_in_view(ctx, rows, cols, smax, win, parts, mem):
    """mem: where g and y live -- device, pinned host (the fused kernel stores y straight into it) or
    pageable host memory."""
    if parts > rows:
        pytest.skip("parts > rows is rejected")
    g = capi.make_phantom(rows, cols, 8, 20.0, 0.5, rows + cols)
    gfull, gv = guarded(rows, cols, dev=mem, init=g)
    yfull, yv = guarded(rows, cols, dev=mem)
    st = capi.lib.hyb_hybrid_u8(ctx.ptr, gv.data_ptr(), gv.stride(0), rows, cols, smax, win, parts,
                                yv.data_ptr(), yv.stride(0), None)
    run(st, ctx, "hybrid")
    ref_y, _ = oracle.hybrid(g, smax, win)
    np.testing.assert_array_equal(yv.cpu().numpy(), ref_y)
    assert_guards(yfull, rows, cols, "hybrid output")
    assert_guards(gfull, rows, cols, "hybrid input")
    np.testing.assert_array_equal(gv.cpu().numpy(), g)


@pytest.mark.parametrize("smax,rb,re", [(7, 0, 700), (9, 13, 611), (11, 650, 700), (15, 0, 1)])
def test_amf_writes_stay_in_view(ctx, smax, rb, re):
    rows, cols = 700, 900
    g = capi.make_phantom(rows, cols, 10, 20.0, 0.5, smax)
    gfull, gv = guarded(rows, cols, init=g)
    ofull, ov = guarded(re - rb, cols)
    ffull, fv = guarded(re - rb, cols)
    st = capi.lib.hyb_amf_u8(ctx.ptr, gv.data_ptr(), gv.stride(0), rows, cols, rb, re, smax,
                             ov.data_ptr(), ov.stride(0), fv.data_ptr(), fv.stride(0))
    run(st, ctx, "amf")
    ref_out, ref_fin = oracle.amf(g, smax, rb, re, finalized_at=True)
    np.testing.assert_array_equal(ov.cpu().numpy(), ref_out)
    np.testing.assert_array_equal(fv.cpu().numpy(), ref_fin)
    assert_guards(ofull, re - rb, cols, "amf output")
    assert_guards(ffull, re - rb, cols, "finalized_at")
    assert_guards(gfull, rows, cols, "amf input")


@pytest.mark.parametrize("win", [1, 3, 5, 7, 9])
def test_wiener_writes_stay_in_view(ctx, win):
    rows, cols = 517, 1031
    f = oracle.amf(capi.make_phantom(rows, cols, 10, 15.0, 0.2, win), 7)
    ffull, fv = guarded(rows, cols, init=f)
    yfull, yv = guarded(rows, cols)
    w = ctypes.c_int64(0)
    st = capi.lib.hyb_wiener_u8(ctx.ptr, fv.data_ptr(), fv.stride(0), rows, cols, win, yv.data_ptr(), yv.stride(0),
                                ctypes.byref(w))
    run(st, ctx, "wiener")
    ref_y, ref_w = oracle.wiener(f, win)
    assert w.value == ref_w
    np.testing.assert_array_equal(yv.cpu().numpy(), ref_y)
    assert_guards(yfull, rows, cols, "wiener output")
    assert_guards(ffull, rows, cols, "wiener input")


@pytest.mark.parametrize("host", [False, True], ids=["device", "host"])
def test_batch_writes_stay_in_slices(ctx, host):
    n, rows, cols = 5, 200, 300
    gap = 2  # canary rows between slices
    stack = np.stack([capi.make_phantom(rows, cols, 6, 20.0, 0.5, s) for s in range(n)])
    dev = "cpu" if host else "cuda"

    def stacked(init=None):
        full = torch.full((n * (rows + gap) + gap, LPAD + cols + RPAD), CANARY, dtype=torch.uint8, device=dev)
        if host:
            full = full.pin_memory()
        views = [full[gap + s * (rows + gap):gap + s * (rows + gap) + rows, LPAD:LPAD + cols] for s in range(n)]
        if init is not None:
            for s in range(n):
                views[s].copy_(torch.from_numpy(init[s]))
        return full, views

    gfull, gvs = stacked(stack)
    yfull, yvs = stacked()
    pitch = gvs[0].stride(0)
    sstride = (rows + gap) * pitch
    w = (ctypes.c_int64 * n)()
    st = capi.lib.hyb_hybrid_batch_u8(ctx.ptr, gvs[0].data_ptr(), pitch, sstride, n, rows, cols, 11, 7,
                                      yvs[0].data_ptr(), pitch, sstride, w)
    run(st, ctx, "batch")
    inside = torch.zeros_like(yfull, dtype=torch.bool)
    for s in range(n):
        ref_y, ref_w = oracle.hybrid(stack[s], 11, 7)
        assert w[s] == ref_w
        np.testing.assert_array_equal(yvs[s].cpu().numpy(), ref_y, err_msg=f"slice {s}")
        inside[gap + s * (rows + gap):gap + s * (rows + gap) + rows, LPAD:LPAD + cols] = True
    assert int((yfull[~inside] != CANARY).sum()) == 0, "batch output: bytes outside the slices were written"
    assert int((gfull[~inside] != CANARY).sum()) == 0, "batch input modified outside the slices"
