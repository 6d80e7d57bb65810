import sys, numpy as np, torch
sys.path.insert(0, ".")
import oracle
from paper_2005_05371_b200 import CONFIGS, capi, denoise
c = CONFIGS[4]; rows, cols, smax = c["rows"], c["cols"], c["smax"]
g = capi.make_phantom(rows, cols, c["ellipses"], c["sigma"], c["density"], 0)
ctx = capi.Context(0)
gd = torch.from_numpy(g).cuda()
f = denoise.adaptive_median_serial(gd, smax, ctx=ctx).cpu().numpy()
f2 = denoise.adaptive_median_serial(gd, smax, ctx=ctx).cpu().numpy()
print("repeat identical:", np.array_equal(f, f2), int((f != f2).sum()))
for a, b in [(0, 192), (rows // 2 - 96, rows // 2 + 96), (rows - 192, rows)]:
    ref, fin = oracle.amf(g, smax, a, b, finalized_at=True)
    bad = np.argwhere(f[a:b] != ref)
    print(f"band [{a},{b}): mismatches {len(bad)}")
    for r, cc in bad[:10]:
        print("   row", a + r, "col", cc, "gpu", f[a + r, cc], "ref", ref[r, cc], "fin", fin[r, cc], "g", g[a + r, cc])
    if len(bad):
        ks = fin[f[a:b] != ref]
        print("   finalized_at of mismatches:", np.unique(ks, return_counts=True))
# smaller crops through the same GPU path
for sz in (4096, 8192):
    sub = np.ascontiguousarray(g[:sz, :sz])
    fs = denoise.adaptive_median_serial(torch.from_numpy(sub).cuda(), smax, ctx=ctx).cpu().numpy()
    ref = oracle.amf(sub, smax, 0, 256)
    print("crop", sz, "top band mismatches", int((fs[:256] != ref).sum()))
