"""B200-native (sm_100a) hybrid adaptive-median + local-Wiener denoiser (arXiv 2005.05371).

The product is libhybrid_cuda.so (C ABI in include/hybrid_cuda.h); this package is its Python
host side: ``capi`` (ctypes binding), ``denoise`` (mirror of the reference's filter API) and
``partition`` (one-process-per-GPU strip partitioner over torch.distributed).
"""
from .capi import CudaError, InvalidArgument, make_phantom  # noqa: F401
from .denoise import (  # noqa: F401
    FilterConfig, HybridResult, adaptive_median_parallel, adaptive_median_rows,
    adaptive_median_serial, hybrid_denoise, hybrid_denoise_batch, split_bands, validate_config,
    validate_smax, wiener_local, window_stats, WindowStats,
)

from .configs import CONFIGS  # noqa: F401  (BASELINE.json configs)
