"""B200-native (sm_100a) hybrid adaptive-median + local-Wiener denoiser (arXiv 2005.05371).

The product is libhybrid_cuda.so (C ABI in include/hybrid_cuda.h); this package is its Python
host side: ``capi`` (ctypes binding), ``denoise`` (mirror of the reference's filter API) and
``partition`` (one-process-per-GPU strip partitioner over torch.distributed).
"""
from .capi import CudaError, InvalidArgument, make_phantom  # noqa: F401
from .denoise import (  # noqa: F401
    FilterConfig, HybridResult, adaptive_median_parallel, adaptive_median_rows,
    adaptive_median_serial, hybrid_denoise, hybrid_denoise_batch, split_bands, validate_config,
    validate_smax, wiener_local,
)

# BASELINE.json configs: (rows, cols, n_ellipses, sigma, density, smax, win, slices)
CONFIGS = {
    0: dict(rows=512, cols=512, ellipses=12, sigma=10.0, density=0.10, smax=7, win=3, slices=1),
    1: dict(rows=1600, cols=1600, ellipses=12, sigma=15.0, density=0.20, smax=7, win=3, slices=1),
    2: dict(rows=8192, cols=8192, ellipses=64, sigma=10.0, density=0.30, smax=9, win=5, slices=1),
    3: dict(rows=512, cols=512, ellipses=12, sigma=8.0, density=0.05, smax=7, win=3, slices=512),
    4: dict(rows=16384, cols=16384, ellipses=256, sigma=20.0, density=0.50, smax=11, win=7, slices=1),
}
