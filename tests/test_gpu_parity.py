"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

AMF: bit-exact (BASELINE.json north_star).  W1 Wiener: the kernel computes the exact rational
result (fp32 with an exact int128 tie check), so it is held to bit-exactness too -- stricter than
the north_star tolerance (<= 1 LSB, >= 99.99 % exact), which is asserted as well.
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle
from paper_2005_05371_b200 import CONFIGS, FilterConfig, capi, denoise

pytestmark = pytest.mark.gpu


def rand_u8(rows, cols, seed, sp=0.0):
    rng = np.random.default_rng(seed)
    img = rng.integers(0, 256, size=(rows, cols), dtype=np.uint8)
    if sp:
        u = rng.random((rows, cols))
        img[u < sp / 2] = 0
        img[(u >= sp / 2) & (u < sp)] = 255
    return img


def wiener_tolerance(y, ref):
    d = np.abs(y.astype(np.int16) - ref.astype(np.int16))
    assert d.max() <= 1
    assert (d == 0).mean() >= 0.9999


# ---------------------------------------------------------------- AMF

def test_amf_kat_ramp(ctx):
    # reference proj/tests/test_adaptive_median.cpp:26-38 (rank-compressed: 0.1..0.9 -> 1..9)
    img = np.arange(1, 10, dtype=np.uint8).reshape(3, 3)
    out = denoise.adaptive_median_serial(img, 3)
    np.testing.assert_array_equal(out, oracle.amf(img, 3))


def test_amf_kat_impulse_on_gradient(ctx):
    # reference proj/tests/test_adaptive_median.cpp:67-78 (0.1(r+c)+0.1 -> r+c+1, salt -> 255)
    img = np.fromfunction(lambda r, c: r + c + 1, (5, 5)).astype(np.uint8)
    img[2, 2] = 255
    out = denoise.adaptive_median_serial(img, 3)
    assert out[2, 2] == 5
    assert out[1, 2] == img[1, 2] and out[3, 1] == img[3, 1]


def test_amf_constant_fixed_point(ctx):
    img = np.full((9, 9), 178, np.uint8)
    np.testing.assert_array_equal(denoise.adaptive_median_serial(img, 11), img)


@pytest.mark.parametrize("smax", [3, 5, 7, 9, 11, 13, 15])
def test_amf_random_vs_oracle(ctx, smax):
    # oracle equivalence (reference proj/tests/test_adaptive_median.cpp:80-96), quantised images
    for trial in range(12):
        rng = np.random.default_rng(1000 + trial)
        rows, cols = int(rng.integers(8, 200)), int(rng.integers(8, 300))
        img = rand_u8(rows, cols, trial, sp=0.2 if trial % 2 == 0 else 0.45)
        out, fin = denoise.adaptive_median_rows(img, smax, 0, rows, finalized_at=True)
        ref_out, ref_fin = oracle.amf(img, smax, finalized_at=True)
        np.testing.assert_array_equal(out, ref_out)
        np.testing.assert_array_equal(fin, ref_fin)


def test_amf_matches_reference_itself(ctx):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    img = rand_u8(63, 57, 5, sp=0.3)
    for smax in (3, 7, 11):
        np.testing.assert_array_equal(denoise.adaptive_median_serial(img, smax), oracle.ref_amf_rows(img, smax))


def test_amf_row_ranges(ctx):
    img = rand_u8(97, 131, 9, sp=0.4)
    for rb, re in [(0, 1), (5, 40), (96, 97), (30, 97), (0, 97)]:
        np.testing.assert_array_equal(denoise.adaptive_median_rows(img, 9, rb, re),
                                      oracle.amf(img, 9, rb, re))


def test_amf_parallel_partition_invariance(ctx):
    # reference proj/tests/test_parallel.cpp:54-76
    img = rand_u8(64, 64, 3, sp=0.25)
    for smax in (3, 11):
        serial = denoise.adaptive_median_serial(img, smax)
        for parts in (2, 3, 4, 8):
            out = denoise.adaptive_median_parallel(img, FilterConfig(smax=smax, parts=parts, workers=4))
            np.testing.assert_array_equal(out, serial)
    odd = rand_u8(63, 57, 4, sp=0.25)
    for parts in (2, 5, 6, 13, 63):
        np.testing.assert_array_equal(denoise.adaptive_median_parallel(odd, FilterConfig(smax=7, parts=parts)),
                                      oracle.amf(odd, 7))


def test_amf_device_tensors(ctx):
    import torch
    img = rand_u8(300, 517, 11, sp=0.3)
    g = torch.from_numpy(img).cuda()
    out = denoise.adaptive_median_serial(g, 7)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), oracle.amf(img, 7))


@pytest.mark.parametrize("cfg", [0, 1, 3])
def test_amf_baseline_configs(ctx, cfg):
    c = CONFIGS[cfg]
    img = capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)
    np.testing.assert_array_equal(denoise.adaptive_median_serial(img, c["smax"]), oracle.amf(img, c["smax"]))


def test_amf_repeated_calls_keep_workspace_consistent(ctx):
    # the growth stage's device counters (tile claims, failure records) must come back to zero after
    # every launch: alternate smax and sizes on one context with device buffers
    c = CONFIGS[1]
    img = capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)
    small = np.ascontiguousarray(img[:300, :700])
    g, gs = torch.from_numpy(img).cuda(), torch.from_numpy(small).cuda()
    want = {s: oracle.amf(img, s) for s in (3, 7, 11)}
    want_small = oracle.amf(small, 7)
    for rep in range(2):
        for smax in (7, 3, 11):
            out = denoise.adaptive_median_serial(g, smax)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(out.cpu().numpy(), want[smax], err_msg=f"rep {rep} smax {smax}")
        out = denoise.adaptive_median_serial(gs, 7)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(out.cpu().numpy(), want_small, err_msg=f"rep {rep} small")


def test_hybrid_fused_launch_modes_agree(ctx):
    # config 1 runs the fused single-kernel step: cooperative (default) and exclusive-device launches,
    # repeated on one context (graph replay in exclusive mode), all equal to the oracle
    c = CONFIGS[1]
    img = capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)
    ref_y, ref_w = oracle.hybrid(img, c["smax"], c["win"])
    g = torch.from_numpy(img).cuda()
    y = torch.empty_like(g)
    for exclusive in (False, True, False):
        ctx.set_exclusive(exclusive)
        for _ in range(3):
            y.fill_(0)
            torch.cuda.synchronize()
            capi.check(capi.lib.hyb_hybrid_u8(ctx.ptr, g.data_ptr(), c["cols"], c["rows"], c["cols"], c["smax"],
                                              c["win"], 1, y.data_ptr(), c["cols"], None), ctx.ptr)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(y.cpu().numpy(), ref_y, err_msg=f"exclusive={exclusive}")
    ctx.set_exclusive(False)
    res = denoise.hybrid_denoise(img, FilterConfig(smax=c["smax"], wiener_window=c["win"]), ctx=ctx)
    assert res.noise_sum == ref_w and res.t_adaptive > 0 and res.t_wiener > 0


def test_amf_worst_case_growth(ctx):
    # config-4 statistics (sigma 20, density 0.5, smax 11) on a 1024^2 crop-sized phantom
    img = capi.make_phantom(1024, 1024, 16, 20.0, 0.5, 0)
    out, fin = denoise.adaptive_median_rows(img, 11, 0, 1024, finalized_at=True)
    ref_out, ref_fin = oracle.amf(img, 11, finalized_at=True)
    np.testing.assert_array_equal(out, ref_out)
    np.testing.assert_array_equal(fin, ref_fin)


def test_amf_wide_growth_row_ranges_and_stacks(ctx):
    """smax 11 on dense impulses takes the wide growth variant with its dynamically claimed last quarter
    of the work (amf.cu GrowWide): row ranges of a source (tiles offset by row_begin) and stacks (tiles
    across slices) against the oracle, finalized_at included."""
    img = capi.make_phantom(700, 900, 16, 20.0, 0.5, 3)
    for rb, re in [(0, 700), (123, 611), (650, 700)]:
        out, fin = denoise.adaptive_median_rows(img, 11, rb, re, finalized_at=True)
        ref_out, ref_fin = oracle.amf(img, 11, rb, re, finalized_at=True)
        np.testing.assert_array_equal(out, ref_out, err_msg=f"rows [{rb},{re})")
        np.testing.assert_array_equal(fin, ref_fin, err_msg=f"rows [{rb},{re})")
    stack = np.stack([capi.make_phantom(384, 512, 10, 20.0, 0.5, s) for s in range(4)])
    y, ws = denoise.hybrid_denoise_batch(stack, 11, 7)
    for s in range(4):
        ref_y, ref_w = oracle.hybrid(stack[s], 11, 7)
        assert ws[s] == ref_w
        np.testing.assert_array_equal(y[s], ref_y, err_msg=f"slice {s}")


# ---------------------------------------------------------------- W1 Wiener

@pytest.mark.parametrize("win", [1, 3, 5, 7, 9])
def test_wiener_vs_oracle(ctx, win):
    for trial in range(6):
        rng = np.random.default_rng(50 + trial)
        rows, cols = int(rng.integers(1, 150)), int(rng.integers(1, 260))
        f = rand_u8(rows, cols, 70 + trial)
        y, w = denoise.wiener_local(f, win)
        ref_y, ref_w = oracle.wiener(f, win)
        assert w == ref_w
        wiener_tolerance(y, ref_y)
        np.testing.assert_array_equal(y, ref_y)


def test_wiener_constant_identity(ctx):
    f = np.full((40, 70), 91, np.uint8)
    y, w = denoise.wiener_local(f, 5)
    assert w == 0
    np.testing.assert_array_equal(y, f)


# ---------------------------------------------------------------- hybrid

@pytest.mark.parametrize("cfg", [0, 1])
def test_hybrid_baseline_configs(ctx, cfg):
    c = CONFIGS[cfg]
    g = capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)
    res = denoise.hybrid_denoise(g, FilterConfig(smax=c["smax"], wiener_window=c["win"]))
    ref_y, ref_w = oracle.hybrid(g, c["smax"], c["win"])
    assert res.noise_sum == ref_w
    wiener_tolerance(res.image, ref_y)
    np.testing.assert_array_equal(res.image, ref_y)


@pytest.mark.parametrize("smax,win", [(9, 5), (11, 7)])
def test_hybrid_large_windows(ctx, smax, win):
    g = capi.make_phantom(700, 900, 20, 20.0, 0.5, 3)
    res = denoise.hybrid_denoise(g, FilterConfig(smax=smax, wiener_window=win))
    ref_y, ref_w = oracle.hybrid(g, smax, win)
    assert res.noise_sum == ref_w
    np.testing.assert_array_equal(res.image, ref_y)


def test_hybrid_strip_invariance(ctx):
    # strips as independent sub-launches with real halo copies == one strip
    g = capi.make_phantom(401, 333, 12, 15.0, 0.2, 7)
    base = denoise.hybrid_denoise(g, FilterConfig(smax=7, wiener_window=3))
    for parts in (2, 3, 4, 5, 8, 13):
        r = denoise.hybrid_denoise(g, FilterConfig(smax=7, parts=parts, wiener_window=3))
        assert r.noise_sum == base.noise_sum
        np.testing.assert_array_equal(r.image, base.image)


def test_hybrid_batch_matches_per_slice(ctx):
    c = CONFIGS[3]
    stack = np.stack([capi.make_phantom(128, 160, 6, c["sigma"], c["density"], s) for s in range(5)])
    y, ws = denoise.hybrid_denoise_batch(stack, c["smax"], c["win"])
    for s in range(5):
        ref_y, ref_w = oracle.hybrid(stack[s], c["smax"], c["win"])
        assert ws[s] == ref_w
        np.testing.assert_array_equal(y[s], ref_y)


def test_hybrid_batch_pipelined_host_buffers(ctx):
    """Host stacks larger than one ~8 MB chunk take the three-stream pipelined path (H2D / hybrid /
    D2H per chunk): same output and per-slice W as the oracle, pageable and pinned buffers."""
    import torch
    c = CONFIGS[3]
    n = 40  # 512 x 512 slices: chunks of 32 -> 2 chunks
    stack = np.stack([capi.make_phantom(512, 512, 12, c["sigma"], c["density"], s) for s in range(n)])
    y, ws = denoise.hybrid_denoise_batch(stack, c["smax"], c["win"])
    refs = [oracle.hybrid(stack[s], c["smax"], c["win"]) for s in range(n)]
    for s in range(n):
        assert ws[s] == refs[s][1]
        np.testing.assert_array_equal(y[s], refs[s][0])
    h_in = torch.from_numpy(stack).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    w = (ctypes.c_int64 * n)()
    capi.check(capi.lib.hyb_hybrid_batch_u8(ctx.ptr, h_in.data_ptr(), 512, 512 * 512, n, 512, 512, c["smax"], c["win"],
                                            h_out.data_ptr(), 512, 512 * 512, w), ctx.ptr)
    for s in range(n):
        assert w[s] == refs[s][1]
        np.testing.assert_array_equal(h_out[s].numpy(), refs[s][0])


def test_mirror_calls_are_ordered_with_torch_streams(ctx):
    """Device-pointer calls are stream-ordered on the context stream; the Python mirror binds it to
    torch's current stream, so torch ops before and after a call see its inputs / outputs (found by the
    config-4 full-size test: an unordered .cpu() read f while the growth kernel still wrote it)."""
    c = CONFIGS[4]
    g = capi.make_phantom(2048, 2048, 32, c["sigma"], c["density"], 5)
    want = oracle.amf(g, c["smax"])
    h = torch.from_numpy(g).pin_memory()
    for stream in (torch.cuda.current_stream(), torch.cuda.Stream()):
        with torch.cuda.stream(stream):
            for rep in range(3):
                gd = torch.empty((2048, 2048), dtype=torch.uint8, device="cuda")
                gd.copy_(h, non_blocking=True)  # input produced on the torch stream
                out = denoise.adaptive_median_serial(gd, c["smax"], ctx=ctx)
                np.testing.assert_array_equal(out.cpu().numpy(), want, err_msg=f"rep {rep}")


# ---------------------------------------------------------------- errors

def test_errors_match_reference_text(ctx):
    img = rand_u8(8, 8, 1)
    with pytest.raises(capi.InvalidArgument, match="odd integer > 1"):
        denoise.adaptive_median_rows(img, 4, 0, 8)
    with pytest.raises(capi.InvalidArgument, match="bad row range"):
        denoise.adaptive_median_rows(img, 3, 5, 3)
    with pytest.raises(capi.InvalidArgument, match="exceeds image rows"):
        denoise.hybrid_denoise(img, FilterConfig(smax=3, parts=9))


# ---------------------------------------------------------------- contrast_stretch

@pytest.mark.parametrize("shape", [(1, 1), (7, 13), (300, 517), (1600, 1600), (33, 4096 + 3)])
def test_contrast_stretch_vs_oracle(ctx, shape):
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    img = rng.integers(31, 190, size=shape, dtype=np.uint8)
    np.testing.assert_array_equal(denoise.contrast_stretch(img), oracle.contrast_stretch(img))
    g = torch.from_numpy(img).cuda()  # device buffers, in place
    denoise.contrast_stretch(g)
    capi.check(capi.lib.hyb_contrast_stretch_u8(ctx.ptr, g.data_ptr(), shape[1], shape[0], shape[1], g.data_ptr(),
                                                shape[1]), ctx.ptr)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(g.cpu().numpy(), oracle.contrast_stretch(img))


def test_contrast_stretch_constant_and_strided(ctx):
    flat = np.full((40, 70), 99, np.uint8)
    np.testing.assert_array_equal(denoise.contrast_stretch(flat), flat)
    base = np.random.default_rng(5).integers(0, 256, size=(50, 100), dtype=np.uint8)
    view = base[3:45, 7:90]  # non-contiguous host view (pitch 100)
    np.testing.assert_array_equal(denoise.contrast_stretch(view), oracle.contrast_stretch(np.ascontiguousarray(view)))


@pytest.mark.parametrize("cfg", [0, 1])
def test_hybrid_stretched_vs_oracle(ctx, cfg):
    c = CONFIGS[cfg]
    g = capi.make_phantom(c["rows"], c["cols"], c["ellipses"], c["sigma"], c["density"], 0)
    res = denoise.hybrid_denoise_stretched(g, FilterConfig(smax=c["smax"], wiener_window=c["win"]))
    ref_y, ref_w = oracle.hybrid(g, c["smax"], c["win"])
    assert res.noise_sum == ref_w
    np.testing.assert_array_equal(res.image, oracle.contrast_stretch(ref_y))


@pytest.mark.parametrize("shape", [(1, 1), (1, 300), (300, 1), (2, 2), (33, 129), (127, 255), (64, 64)])
@pytest.mark.parametrize("smax,win", [(3, 1), (5, 3), (7, 5), (11, 7), (13, 3), (7, 9)])
def test_hybrid_small_shapes_vs_oracle(ctx, shape, smax, win):
    # small images take the fused single-kernel path (smax <= 11, win <= 7) or the separate kernels
    # otherwise; both must equal the oracle, including degenerate 1-pixel-wide images
    rng = np.random.default_rng(shape[0] * 1000 + shape[1] + smax * 7 + win)
    g = rng.integers(0, 256, size=shape, dtype=np.uint8)
    g[rng.random(shape) < 0.25] = 0
    res = denoise.hybrid_denoise(g, FilterConfig(smax=smax, wiener_window=win))
    ref_y, ref_w = oracle.hybrid(g, smax, win)
    assert res.noise_sum == ref_w
    np.testing.assert_array_equal(res.image, ref_y)
    gd = torch.from_numpy(g).cuda()
    yd = torch.empty_like(gd)
    capi.check(capi.lib.hyb_hybrid_u8(ctx.ptr, gd.data_ptr(), shape[1], shape[0], shape[1], smax, win, 1,
                                      yd.data_ptr(), shape[1], None), ctx.ptr)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(yd.cpu().numpy(), ref_y)
