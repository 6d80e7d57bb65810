"""Extended randomized parity run of the wide AMF growth variant (smax >= 11, bit-plane levels) against the
oracle: random shapes, densities (salt / pepper mixes), row ranges, finalized_at.  usage: fuzz_wide.py [cases] [seed]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2005_05371_b200 import capi, denoise  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 12345)
t0 = time.time()
for n in range(cases):
    rows, cols = int(rng.integers(1, 900)), int(rng.integers(1, 1100))
    smax = int(rng.choice([11, 11, 11, 13, 15, 17]))
    d = float(rng.choice([0.0, 0.1, 0.3, 0.5, 0.5, 0.7, 0.9, 0.97]))
    salt = float(rng.choice([0.0, 0.5, 0.5, 1.0, 0.2]))  # share of the impulses that are 255
    kind = int(rng.integers(0, 3))
    if kind == 0:
        base = rng.integers(0, 256, size=(rows, cols), dtype=np.uint8)
    elif kind == 1:
        base = capi.make_phantom(rows, cols, 4, 15.0, 0.0, int(rng.integers(0, 10**6)))
    else:
        base = np.full((rows, cols), int(rng.choice([0, 1, 100, 254, 255])), np.uint8)
    u, v = rng.random((rows, cols)), rng.random((rows, cols))
    g = base.copy()
    g[(u < d) & (v < salt)] = 255
    g[(u < d) & (v >= salt)] = 0
    gd = torch.from_numpy(g).cuda()
    a = int(rng.integers(0, rows))
    b = int(rng.integers(a + 1, rows + 1))
    fin = bool(rng.integers(0, 2))
    if fin:
        f, fa = denoise.adaptive_median_rows(gd, smax, a, b, finalized_at=True)
        rf, rfa = oracle.amf(g, smax, a, b, finalized_at=True)
        assert np.array_equal(fa.cpu().numpy(), rfa), ("fin", n, rows, cols, smax, d, salt, kind, a, b)
    else:
        f = denoise.adaptive_median_rows(gd, smax, a, b)
        rf = oracle.amf(g, smax, a, b)
    assert np.array_equal(f.cpu().numpy(), rf), (n, rows, cols, smax, d, salt, kind, a, b)
print(f"ok {cases} cases in {time.time() - t0:.0f} s")
