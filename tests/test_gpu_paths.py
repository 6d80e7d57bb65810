"""Both AMF kernel paths against the oracle, whichever the dispatch picks by default: the two-kernel path
(amf_k3_kernel + amf_grow_kernel) and the fused per-batch
kernel (amf_fused_kernel), forced by HYB_AMF_SPLIT / HYB_AMF_FUSED in a subprocess (the library reads
them once).  Row ranges, finalized_at, stacks, borders and every smax variant of both."""
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
rng = np.random.default_rng(5)
n = 0
for smax in (5, 7, 9, 11, 13, 15):
    for (rows, cols, sp) in ((333, 517, 0.5), (130, 260, 0.2), (1000, 700, 0.35), (40, 33, 0.9)):
        g = capi.make_phantom(rows, cols, 6, 15.0, sp, smax * 7 + rows)
        gd = torch.from_numpy(g).cuda()
        f, fin = denoise.adaptive_median_rows(gd, smax, 0, rows, finalized_at=True)
        rf, rfin = oracle.amf(g, smax, finalized_at=True)
        assert np.array_equal(f.cpu().numpy(), rf), (smax, rows, cols)
        assert np.array_equal(fin.cpu().numpy(), rfin), (smax, rows, cols, "fin")
        a, b = rows // 3, rows // 3 + rows // 4 + 1
        f2 = denoise.adaptive_median_rows(gd, smax, a, b)
        assert np.array_equal(f2.cpu().numpy(), oracle.amf(g, smax, a, b)), (smax, "range")
        n += 3
    stack = np.stack([capi.make_phantom(96, 160, 5, 10.0, 0.4, s) for s in range(9)])
    y, ws = denoise.hybrid_denoise_batch(torch.from_numpy(stack).cuda(), smax, 5)
    y = y.cpu().numpy()
    for s in range(9):
        ry, rw = oracle.hybrid(stack[s], smax, 5)
        assert ws[s] == rw and np.array_equal(y[s], ry), (smax, "stack", s)
    n += 9
print("ok", n)
'''


@pytest.mark.parametrize("env", ["HYB_AMF_SPLIT", "HYB_AMF_FUSED", "HYB_FUSED_LEAN11"])
def test_amf_paths_vs_oracle(env):
    e = dict(os.environ)
    e[env] = "1"
    if env == "HYB_FUSED_LEAN11":
        e["HYB_AMF_FUSED"] = "1"
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.strip().startswith("ok"), r.stdout
