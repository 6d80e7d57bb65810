"""BASELINE.json configs (pure Python, no native code: bench.py's CPU reference arm reads this file
without importing the package, so it never maps libhybrid_cuda.so).

Each entry: rows, cols, ellipses, sigma, density (S&P), smax (AMF), win (Wiener), slices.
"""

CONFIGS = {
    0: dict(rows=512, cols=512, ellipses=12, sigma=10.0, density=0.10, smax=7, win=3, slices=1),
    1: dict(rows=1600, cols=1600, ellipses=12, sigma=15.0, density=0.20, smax=7, win=3, slices=1),
    2: dict(rows=8192, cols=8192, ellipses=64, sigma=10.0, density=0.30, smax=9, win=5, slices=1),
    3: dict(rows=512, cols=512, ellipses=12, sigma=8.0, density=0.05, smax=7, win=3, slices=512),
    4: dict(rows=16384, cols=16384, ellipses=256, sigma=20.0, density=0.50, smax=11, win=7, slices=1),
}
