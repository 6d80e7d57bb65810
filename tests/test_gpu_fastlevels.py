"""The bit-plane growth levels of the wide AMF variant (smax >= 11; amf_core.cuh grow_levels_fast) against the
oracle on the inputs that steer pixels through each of its routes: heavy salt & pepper (plane tests decide),
images with no 0 or no 255 (every growing pixel flagged: the generic test in the median passes), salt only /
pepper only, all-impulse and constant images, mixed halves, segments split across batches, row ranges and
finalized_at; and the same inputs on the plain levels (HYB_GROW_FAST=0, read once per process)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
from paper_2005_05371_b200 import capi, denoise

def inputs(rows, cols, seed):
    rng = np.random.default_rng(seed)
    base = capi.make_phantom(rows, cols, 5, 12.0, 0.0, seed)           # no impulses
    u = rng.random((rows, cols))
    yield "s&p 0.5", capi.make_phantom(rows, cols, 5, 20.0, 0.5, seed)
    yield "s&p 0.7", capi.make_phantom(rows, cols, 5, 20.0, 0.7, seed + 1)
    yield "pepper only", np.where(u < 0.45, 0, np.clip(base, 1, 254)).astype(np.uint8)
    yield "salt only", np.where(u < 0.45, 255, np.clip(base, 1, 254)).astype(np.uint8)
    yield "two-level 0/200", np.where(u < 0.5, 0, 200).astype(np.uint8)
    yield "two-level 0/255", np.where(u < 0.5, 0, 255).astype(np.uint8)
    yield "constant 0", np.zeros((rows, cols), np.uint8)
    yield "constant 255", np.full((rows, cols), 255, np.uint8)
    yield "constant 100", np.full((rows, cols), 100, np.uint8)
    half = capi.make_phantom(rows, cols, 5, 20.0, 0.6, seed + 2)
    half[:, cols // 2:] = np.clip(base[:, cols // 2:], 1, 254)           # right half: nothing to grow
    yield "half s&p", half
    blocks = capi.make_phantom(rows, cols, 5, 20.0, 0.5, seed + 3)
    blocks[rows // 4: rows // 2, :] = 0                                    # a black band: windows without a 255
    blocks[:, cols // 3: cols // 3 + 9] = 255                              # a white stripe
    yield "bands", blocks

n = 0
for smax in (11, 13, 15):
    for (rows, cols) in ((257, 300), (64, 1000), (97, 131)):
        for name, g in inputs(rows, cols, smax * 100 + rows):
            gd = torch.from_numpy(np.ascontiguousarray(g)).cuda()
            f, fin = denoise.adaptive_median_rows(gd, smax, 0, rows, finalized_at=True)
            rf, rfin = oracle.amf(g, smax, finalized_at=True)
            assert np.array_equal(f.cpu().numpy(), rf), (smax, rows, cols, name)
            assert np.array_equal(fin.cpu().numpy(), rfin), (smax, rows, cols, name, "fin")
            f1 = denoise.adaptive_median_rows(gd, smax, 0, rows)
            assert np.array_equal(f1.cpu().numpy(), rf), (smax, rows, cols, name, "no fin")
            a, b = rows // 5, rows // 5 + rows // 2 + 3
            f2 = denoise.adaptive_median_rows(gd, smax, a, b)
            assert np.array_equal(f2.cpu().numpy(), oracle.amf(g, smax, a, b)), (smax, name, "range")
            n += 4
# windows beyond the plane tests and the unrolled selects (generic levels), taller halos
for smax in (19, 33):
    for name, g in inputs(150, 200, smax):
        gd = torch.from_numpy(np.ascontiguousarray(g)).cuda()
        f, fin = denoise.adaptive_median_rows(gd, smax, 0, 150, finalized_at=True)
        rf, rfin = oracle.amf(g, smax, finalized_at=True)
        assert np.array_equal(f.cpu().numpy(), rf), (smax, name)
        assert np.array_equal(fin.cpu().numpy(), rfin), (smax, name, "fin")
        n += 1
# many tiles per CTA: segments of one tile split across batches / CTAs
g = capi.make_phantom(2100, 4200, 30, 20.0, 0.5, 77)
gd = torch.from_numpy(g).cuda()
res = denoise.hybrid_denoise(gd, denoise.FilterConfig(smax=11, wiener_window=7))
ry, rw = oracle.hybrid(g, 11, 7)
assert res.noise_sum == rw and np.array_equal(res.image.cpu().numpy(), ry), "large hybrid"
print("ok", n + 1)
'''


@pytest.mark.parametrize("fast", ["1", "0"])
def test_wide_growth_routes_vs_oracle(fast):
    e = dict(os.environ)
    e["HYB_GROW_FAST"] = fast
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.strip().startswith("ok"), r.stdout


def test_wide_growth_randomized():
    """tools/fuzz_wide.py: 250 random shapes / densities / salt-pepper mixes / row ranges at smax 11..17."""
    r = subprocess.run([sys.executable, "tools/fuzz_wide.py", "250", "99"], cwd=ROOT, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.strip().startswith("ok"), r.stdout
