"""Compact growth windows (amf_core.cuh CompactOut): sparse k = 3 strips (at most
HYB_COMPACT_T level-A failures) hand their failures to the growth as 64-byte 7 x 7 window entries
instead of bitmap bits, so the growth never reloads their tiles (smax 5 / 7 on the two-kernel path:
stacks, and single images under HYB_AMF_SPLIT).  Checked bit-exact against the oracle with mixed
sparse / dense strips, borders, row ranges, finalized_at, padded pitches, and with the entry list
forced tiny (HYB_COMPACT_CAP) so strips overflow to the bitmap and straddling reservations are voided."""
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
rng = np.random.default_rng(11)
n = 0
for smax in (5, 7):
    for (rows, cols, sp) in ((333, 517, 0.02), (130, 260, 0.05), (700, 1000, 0.08), (40, 33, 0.03), (257, 129, 0.12)):
        g = capi.make_phantom(rows, cols, 6, 15.0, sp, smax * 13 + rows)
        # a dense band so one image mixes compact and bitmap strips
        band = rng.random((rows // 5, cols)) < 0.5
        g[rows // 3: rows // 3 + rows // 5][band] = rng.choice(np.array([0, 255], np.uint8), int(band.sum()))
        gd = torch.from_numpy(g).cuda()
        f, fin = denoise.adaptive_median_rows(gd, smax, 0, rows, finalized_at=True)
        rf, rfin = oracle.amf(g, smax, finalized_at=True)
        assert np.array_equal(f.cpu().numpy(), rf), (smax, rows, cols, int((f.cpu().numpy() != rf).sum()))
        assert np.array_equal(fin.cpu().numpy(), rfin), (smax, rows, cols, "fin")
        a, b = rows // 4, rows // 4 + rows // 2 + 1
        f2 = denoise.adaptive_median_rows(gd, smax, a, b)
        assert np.array_equal(f2.cpu().numpy(), oracle.amf(g, smax, a, b)), (smax, "range")
        n += 3
    for (rows, cols, ns) in ((96, 160, 9), (512, 512, 6), (33, 517, 4)):
        stack = np.stack([capi.make_phantom(rows, cols, 5, 8.0, 0.02 + 0.03 * s, 100 * smax + s) for s in range(ns)])
        y, ws = denoise.hybrid_denoise_batch(torch.from_numpy(stack).cuda(), smax, 3)
        y = y.cpu().numpy()
        for s in range(ns):
            ry, rw = oracle.hybrid(stack[s], smax, 3)
            assert ws[s] == rw and np.array_equal(y[s], ry), (smax, "stack", rows, cols, s)
        n += ns
    # padded row pitch (device view into a wider buffer)
    g = capi.make_phantom(300, 400, 6, 10.0, 0.04, 7 + smax)
    wide = torch.zeros((300, 448), dtype=torch.uint8, device="cuda")
    wide[:, :400] = torch.from_numpy(g).cuda()
    f = denoise.adaptive_median_rows(wide[:, :400], smax, 0, 300)
    assert np.array_equal(f.cpu().numpy(), oracle.amf(g, smax)), (smax, "pitch")
    n += 1
print("ok", n)
'''


@pytest.mark.parametrize("env", [{}, {"HYB_COMPACT_T": "32"}, {"HYB_COMPACT_T": "1"},
                                 {"HYB_COMPACT_CAP": "37"}, {"HYB_COMPACT_CAP": "1", "HYB_COMPACT_T": "32"},
                                 {"HYB_COMPACT_T": "0"}])
def test_compact_growth_vs_oracle(env):
    e = dict(os.environ)
    e["HYB_AMF_SPLIT"] = "1"
    e.update(env)
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.strip().startswith("ok"), r.stdout
