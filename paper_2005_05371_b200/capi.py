"""ctypes binding of libhybrid_cuda.so (include/hybrid_cuda.h).

The shared library is built in-tree by ``make`` (or ``__graft_entry__.build()``).  There is no
fallback: if the library is missing, importing this module raises, and every entry point
reports CUDA errors as exceptions.  Status codes map onto the reference's exception types
(SURVEY.md 8(b)): HYB_EINVAL -> InvalidArgument (std::invalid_argument), everything else ->
CudaError (std::runtime_error).
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int64, c_size_t, c_uint64, c_void_p

import numpy as np

HYB_OK, HYB_EINVAL, HYB_ECUDA, HYB_ENCCL, HYB_ENOMEM = 0, 1, 2, 3, 4

# HYB_LIB selects a debug build of the same library in this directory (e.g. the `make trace` one)
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                        os.path.basename(os.environ.get("HYB_LIB", "libhybrid_cuda.so")))

# Every symbol include/hybrid_cuda.h declares (checked by tests/test_capi_symbols.py).
EXPORTED = (
    "hyb_create", "hyb_create_multi", "hyb_context_devices", "hyb_destroy", "hyb_set_stream", "hyb_set_exclusive", "hyb_set_async", "hyb_synchronize", "hyb_last_error", "hyb_kernel_launches",
    "hyb_validate_smax", "hyb_validate_config", "hyb_amf_u8", "hyb_amf_batch_u8",
    "hyb_wiener_stats_u8", "hyb_wiener_gain_u8", "hyb_wiener_u8", "hyb_hybrid_u8",
    "hyb_hybrid_batch_u8", "hyb_window_stats_u8", "hyb_contrast_stretch_u8", "hyb_hybrid_stretch_u8",
    "hyb_wiener_freq_f64", "hyb_contrast_stretch_f64", "hyb_noise_robust_f64", "hyb_noise_reference_f64", "hyb_make_phantom_u8",
)


class InvalidArgument(ValueError):
    """Mirror of std::invalid_argument thrown by the reference."""


class CudaError(RuntimeError):
    """CUDA / allocation failure (std::runtime_error)."""


class HybStats(ctypes.Structure):
    _fields_ = [
        ("noise_sum", c_int64),
        ("pixel_count", c_int64),
        ("sigma2", c_double),
        ("t_adaptive", c_double),
        ("t_wiener", c_double),
        ("t_total", c_double),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
            "there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    P, Pi64 = c_void_p, POINTER(c_int64)
    sig = {
        "hyb_create": (c_void_p, [c_int, POINTER(c_int)]),
        "hyb_create_multi": (c_void_p, [c_int, POINTER(c_int), POINTER(c_int)]),
        "hyb_context_devices": (c_int, [P, POINTER(c_int)]),
        "hyb_destroy": (c_int, [P]),
        "hyb_set_stream": (c_int, [P, c_void_p]),
        "hyb_set_exclusive": (c_int, [P, c_int]),
        "hyb_set_async": (c_int, [P, c_int]),
        "hyb_synchronize": (c_int, [P]),
        "hyb_last_error": (c_char_p, [P]),
        "hyb_kernel_launches": (c_int64, [P]),
        "hyb_validate_smax": (c_int, [c_int]),
        "hyb_validate_config": (c_int, [c_int, c_int, c_int]),
        "hyb_amf_u8": (c_int, [P, P, c_size_t, c_int, c_int, c_int, c_int, c_int, P, c_size_t, P, c_size_t]),
        "hyb_amf_batch_u8": (c_int, [P, P, c_size_t, c_size_t, c_int, c_int, c_int, c_int, P, c_size_t, c_size_t]),
        "hyb_wiener_stats_u8": (c_int, [P, P, c_size_t, c_int, c_int, c_int, c_int, c_int, c_void_p]),
        "hyb_wiener_gain_u8": (c_int, [P, P, c_size_t, c_int, c_int, c_int, c_int, c_int, c_void_p, c_int64,
                                       P, c_size_t]),
        "hyb_wiener_u8": (c_int, [P, P, c_size_t, c_int, c_int, c_int, P, c_size_t, Pi64]),
        "hyb_hybrid_u8": (c_int, [P, P, c_size_t, c_int, c_int, c_int, c_int, c_int, P, c_size_t,
                                  POINTER(HybStats)]),
        "hyb_window_stats_u8": (c_int, [P, P, c_size_t, c_int, c_int, c_int, P, P, P, c_size_t]),
        "hyb_hybrid_batch_u8": (c_int, [P, P, c_size_t, c_size_t, c_int, c_int, c_int, c_int, c_int, P,
                                        c_size_t, c_size_t, Pi64]),
        "hyb_contrast_stretch_u8": (c_int, [P, P, c_size_t, c_int, c_int, P, c_size_t]),
        "hyb_hybrid_stretch_u8": (c_int, [P, P, c_size_t, c_int, c_int, c_int, c_int, c_int, P, c_size_t,
                                          POINTER(HybStats)]),
        "hyb_wiener_freq_f64": (c_int, [P, P, c_size_t, c_int, c_int, c_double, c_int, P, c_size_t]),
        "hyb_contrast_stretch_f64": (c_int, [P, P, c_size_t, c_int, c_int, P, c_size_t]),
        "hyb_noise_robust_f64": (c_int, [P, P, c_size_t, c_int, c_int, POINTER(c_double)]),
        "hyb_noise_reference_f64": (c_int, [P, P, c_size_t, P, c_size_t, c_int, c_int, POINTER(c_double)]),
        "hyb_make_phantom_u8": (c_int, [c_int, c_int, c_int, c_double, c_double, c_uint64, P, c_size_t]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int, ctx=None) -> None:
    if status == HYB_OK:
        return
    msg = lib.hyb_last_error(ctx).decode() if ctx else f"status {status}"
    if status == HYB_EINVAL:
        raise InvalidArgument(msg)
    raise CudaError(f"libhybrid_cuda status {status}: {msg}")


class Context:
    """Owns one hyb_ctx (one CUDA device, one stream, pooled device scratch), or with `devices` a
    multi-device context (hyb_create_multi: one strip / slice chunk per listed device)."""

    def __init__(self, device: int = 0, devices=None):
        st = c_int(0)
        if devices is not None:
            ids = (c_int * len(devices))(*devices)
            self.ptr = lib.hyb_create_multi(len(devices), ids, ctypes.byref(st))
            device = devices[0] if devices else device
        else:
            self.ptr = lib.hyb_create(device, ctypes.byref(st))
        if not self.ptr:
            raise CudaError(f"hyb_create(device={device}, devices={devices}) failed with status {st.value} "
                            "(no CUDA device?)")
        self.device = device

    def devices(self) -> list:
        n = lib.hyb_context_devices(self.ptr, None)
        ids = (c_int * n)()
        lib.hyb_context_devices(self.ptr, ids)
        return list(ids)

    def close(self) -> None:
        if self.ptr:
            lib.hyb_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int | None) -> None:
        check(lib.hyb_set_stream(self.ptr, stream_handle), self.ptr)

    def set_exclusive(self, exclusive: bool) -> None:
        """Dedicated-GPU mode (hyb_set_exclusive): plain instead of cooperative fused launches."""
        check(lib.hyb_set_exclusive(self.ptr, int(bool(exclusive))), self.ptr)

    def set_async(self, on: bool) -> None:
        """hyb_set_async: host-buffer calls return once enqueued (double-buffered staging); synchronize()."""
        check(lib.hyb_set_async(self.ptr, int(bool(on))), self.ptr)

    def synchronize(self) -> None:
        check(lib.hyb_synchronize(self.ptr), self.ptr)

    def launches(self) -> int:
        return int(lib.hyb_kernel_launches(self.ptr))


_default: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    ctx = _default.get(device)
    if ctx is None:
        ctx = _default[device] = Context(device)
    return ctx


def buf(a):
    """(pointer, row pitch in bytes) of a 2-D (or 3-D slice stack) uint8 numpy array or torch tensor."""
    if isinstance(a, np.ndarray):
        if a.dtype != np.uint8:
            raise InvalidArgument(f"expected uint8 pixels, got {a.dtype}")
        if a.strides[-1] != 1:
            raise InvalidArgument("rows must be contiguous")
        return a.ctypes.data, a.strides[-2]
    # torch tensor (host or CUDA)
    import torch
    if a.dtype != torch.uint8:
        raise InvalidArgument(f"expected uint8 pixels, got {a.dtype}")
    if a.stride(-1) != 1:
        raise InvalidArgument("rows must be contiguous")
    return a.data_ptr(), a.stride(-2)


def make_phantom(rows: int, cols: int, n_ellipses: int, sigma: float, density: float, seed: int) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.uint8)
    st = lib.hyb_make_phantom_u8(rows, cols, n_ellipses, float(sigma), float(density), seed,
                                 out.ctypes.data, cols)
    if st != HYB_OK:
        raise InvalidArgument(f"bad phantom parameters: {rows}x{cols}, {n_ellipses}, {sigma}, {density}")
    return out
