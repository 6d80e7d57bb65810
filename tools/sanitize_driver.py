"""Small end-to-end driver for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every
kernel family of libhybrid_cuda on images small enough for the sanitizers, each result checked against
the CPU oracle.  usage: compute-sanitizer --tool T python tools/sanitize_driver.py
(compute-sanitizer is closed on this round's GPU pool; tests/test_gpu_guard.py checks for stray writes
with canary-filled guard bands instead.)

Covers: the fused small-image kernel (hyb_hybrid_u8 on <= 888 tiles, cooperative and exclusive
launch), the separate k3 -> growth kernels (hyb_amf_u8 with row ranges and finalized_at, lean and wide
growth variants), the W1 statistics / gain kernels (hyb_wiener_u8, windows 3..9), the separate-kernel
hybrid (strips, parts = 2), the batched stack path and contrast stretch.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (checker only)
from paper_2005_05371_b200 import FilterConfig, capi, denoise  # noqa: E402


def eq(a, b, what):
    if not np.array_equal(np.asarray(a), np.asarray(b)):
        raise SystemExit(f"MISMATCH: {what}")
    print("ok", what, flush=True)


def main():
    ctx = capi.default_context(0)
    g = capi.make_phantom(300, 333, 6, 20.0, 0.5, 1)

    # fused kernel (small image), both launch modes
    for excl in (False, True):
        ctx.set_exclusive(excl)
        res = denoise.hybrid_denoise(g, FilterConfig(smax=7, wiener_window=3), ctx=ctx)
        y, w = oracle.hybrid(g, 7, 3)
        eq(res.image, y, f"fused hybrid smax 7 win 3 exclusive={excl}")
        assert res.noise_sum == w
    ctx.set_exclusive(False)
    res = denoise.hybrid_denoise(g, FilterConfig(smax=11, wiener_window=7), ctx=ctx)
    eq(res.image, oracle.hybrid(g, 11, 7)[0], "fused hybrid smax 11 win 7")

    # separate AMF kernels: lean (smax 9) and wide (smax 11) growth, row ranges, finalized_at
    for smax, (rb, re) in [(9, (0, 300)), (11, (17, 251))]:
        out, fin = denoise.adaptive_median_rows(g, smax, rb, re, finalized_at=True, ctx=ctx)
        ref_out, ref_fin = oracle.amf(g, smax, rb, re, finalized_at=True)
        eq(out, ref_out, f"amf smax {smax} rows [{rb},{re})")
        eq(fin, ref_fin, f"amf finalized_at smax {smax}")

    # W1 kernels
    f = oracle.amf(g, 7)
    for win in (3, 5, 7, 9):
        y, w = denoise.wiener_local(f, win, ctx=ctx)
        eq(y, oracle.wiener(f, win)[0], f"wiener win {win}")

    # separate-kernel hybrid over strips
    res = denoise.hybrid_denoise(g, FilterConfig(smax=7, wiener_window=5, parts=2), ctx=ctx)
    eq(res.image, oracle.hybrid(g, 7, 5)[0], "strip hybrid parts 2")

    # batched stack
    stack = np.stack([capi.make_phantom(128, 160, 4, 15.0, 0.3, s) for s in range(3)])
    ys, ws = denoise.hybrid_denoise_batch(stack, 7, 3, ctx=ctx)
    for s in range(3):
        eq(ys[s], oracle.hybrid(stack[s], 7, 3)[0], f"batch slice {s}")

    # contrast stretch
    eq(denoise.contrast_stretch(g, ctx=ctx), oracle.contrast_stretch(g), "contrast stretch")
    print("SANITIZE DRIVER OK", flush=True)


if __name__ == "__main__":
    main()
