"""Host-side mirror of the reference's filter API for the hot path, on libhybrid_cuda.

Same names, argument meaning and error behaviour as the reference's ``namespace denoise``
(proj/include/denoise/{adaptive_median,parallel,tiling,pipeline}.hpp); images are uint8 arrays
(numpy on the host, or torch uint8 tensors on the GPU) instead of ``Image`` doubles -- the
reference's k/255 doubles map onto uint8 exactly for this path (SURVEY.md finding 4;
``to_u8`` / ``to_unit`` below).  Every filter call goes through the C ABI; there is no CPU path.
"""
from __future__ import annotations

import ctypes
import sys
from dataclasses import dataclass

import numpy as np

from . import capi
from .capi import InvalidArgument, check, lib


def _ctx(ctx, *arrays):
    """The context for a call on `arrays`: the caller's, else the default context of the device the
    CUDA tensors live on (device 0 for host arrays).  Inputs on different devices, or on a device
    other than the given context's, are rejected."""
    devs = {a.device.index for a in arrays
            if a is not None and _is_torch(a) and getattr(a, "is_cuda", False)}
    if len(devs) > 1:
        raise InvalidArgument(f"inputs on different CUDA devices: {sorted(devs)}")
    dev = devs.pop() if devs else None
    if ctx is None:
        c = capi.default_context(dev if dev is not None else 0)
    else:
        c = ctx
        if dev is not None and dev != c.device:
            raise InvalidArgument(f"tensor on cuda:{dev} but the context drives device {c.device}")
    _bind_torch_stream(c)
    return c.ptr


def _bind_torch_stream(c) -> None:
    """Device-pointer calls are stream-ordered on the context stream (include/hybrid_cuda.h), so the
    torch-facing mirror runs them on torch's current stream: inputs produced and outputs consumed by
    torch are ordered with the kernels, as the reference's by-value calls are.  torch's default
    stream is the legacy stream (handle 0), passed as cudaStreamLegacy (1)."""
    torch = sys.modules.get("torch")
    if torch is None or not torch.cuda.is_available() or not torch.cuda.is_initialized():
        return
    h = torch.cuda.current_stream(c.device).cuda_stream
    c.set_stream(h if h else 1)


def _is_torch(a) -> bool:
    return not isinstance(a, np.ndarray)


def _empty_like(a, rows, cols):
    if _is_torch(a):
        import torch
        return torch.empty((rows, cols), dtype=torch.uint8, device=a.device)
    return np.empty((rows, cols), dtype=np.uint8)


def _shape(a):
    if a.ndim != 2:
        raise InvalidArgument(f"expected a 2-D image, got {a.ndim} dimensions")
    return int(a.shape[0]), int(a.shape[1])


# ---------------------------------------------------------------- validation

def validate_smax(smax: int) -> None:
    """validate_smax -- reference proj/src/adaptive_median.cpp:11-16."""
    if lib.hyb_validate_smax(int(smax)) != capi.HYB_OK:
        raise InvalidArgument(f"smax must be an odd integer > 1, got {smax}")


class EstimateMode:
    """EstimateMode -- reference proj/include/denoise/wiener.hpp:8.  For the W1 Wiener: ROBUST = the
    north_star's estimator (mean of the local variances, exact int64 W); REFERENCE = the mean squared
    difference between the AMF output and a reference image (proj/src/wiener.cpp:31-42)."""
    ROBUST = "robust"
    REFERENCE = "reference"


@dataclass
class FilterConfig:
    """FilterConfig -- reference proj/include/denoise/parallel.hpp:13-19 (same fields and defaults),
    plus the W1 window and where it runs: `gpus` > 1 strips on devices 0..gpus-1 or an explicit
    `device_ids` list (a multi-device context: one strip per device, bit-identical to one GPU), and
    `final_stretch`, the reference pipeline's closing contrast_stretch (proj/src/pipeline.cpp:55-57)."""
    smax: int = 11
    parts: int = 1
    workers: int = 1
    estimate_mode: str = EstimateMode.ROBUST
    use_halo: bool = True
    wiener_window: int = 3
    gpus: int = 1
    device_ids: tuple = ()
    final_stretch: bool = False


_multi: dict = {}


def _config_ctx(ctx, config, *arrays):
    """The context for a config: the caller's, else a (cached) multi-device context when the config asks
    for several devices, else the inputs' device's default context."""
    if ctx is None:
        ids = tuple(config.device_ids) if config.device_ids else tuple(range(config.gpus))
        if config.gpus < 1:
            raise InvalidArgument(f"gpus must be >= 1, got {config.gpus}")
        if len(ids) > 1:
            ctx = _multi.get(ids)
            if ctx is None:
                ctx = _multi[ids] = capi.Context(devices=list(ids))
    return _ctx(ctx, *arrays)


def validate_config(config: FilterConfig) -> None:
    """validate_config -- reference proj/src/parallel.cpp:16-25."""
    validate_smax(config.smax)
    if config.parts < 1:
        raise InvalidArgument(f"parts must be >= 1, got {config.parts}")
    if config.workers < 1:
        raise InvalidArgument(f"workers must be >= 1, got {config.workers}")


# ---------------------------------------------------------------- tiling

@dataclass
class Band:
    """Tile geometry -- reference proj/include/denoise/tiling.hpp:12-19 (without the pixel copy)."""
    index: int
    core_start: int
    core_rows: int
    halo_above: int
    halo_below: int


def split_bands(rows: int, parts: int, halo: int) -> list[Band]:
    """Band geometry of split_bands -- reference proj/src/tiling.cpp:10-45: heights rows // parts
    with the first rows % parts bands one taller; halos clamped at the image borders."""
    if parts < 1 or parts > rows:
        raise InvalidArgument(f"parts must be in [1, {rows}], got {parts}")
    if halo < 0:
        raise InvalidArgument(f"halo must be nonnegative, got {halo}")
    base, extra = divmod(rows, parts)
    out, start = [], 0
    for i in range(parts):
        core = base + (1 if i < extra else 0)
        out.append(Band(i, start, core, min(halo, start), min(halo, rows - start - core)))
        start += core
    return out


# ---------------------------------------------------------------- AMF

def adaptive_median_rows(src, smax: int, row_begin: int, row_end: int, finalized_at: bool = False,
                         ctx=None):
    """detail::adaptive_median_rows -- reference proj/include/denoise/adaptive_median.hpp:47-48."""
    rows, cols = _shape(src)
    out = _empty_like(src, max(row_end - row_begin, 0), cols)
    fin = _empty_like(src, max(row_end - row_begin, 0), cols) if finalized_at else None
    sp, spitch = capi.buf(src)
    dp, dpitch = capi.buf(out) if out.shape[0] else (0, cols)
    fp, fpitch = capi.buf(fin) if fin is not None and fin.shape[0] else (None, cols)
    c = _ctx(ctx, src, out, fin)
    check(lib.hyb_amf_u8(c, sp, spitch, rows, cols, row_begin, row_end, smax, dp, dpitch, fp, fpitch), c)
    return (out, fin) if finalized_at else out


def adaptive_median_serial(image, smax: int, ctx=None):
    """adaptive_median_serial -- reference proj/src/adaptive_median.cpp:219-224."""
    validate_smax(smax)
    return adaptive_median_rows(image, smax, 0, _shape(image)[0], ctx=ctx)


def adaptive_median_parallel(image, config: FilterConfig, ctx=None):
    """adaptive_median_parallel -- reference proj/src/parallel.cpp:27-70: bands with halo
    (smax-1)/2 (0 without use_halo), each filtered from its own copy, then stitched.  With the
    halo the result is bit-identical to adaptive_median_serial for every parts."""
    validate_config(config)
    rows, cols = _shape(image)
    if config.parts > rows:
        raise InvalidArgument(f"parts {config.parts} exceeds image rows {rows}")
    halo = (config.smax - 1) // 2 if config.use_halo else 0
    out = _empty_like(image, rows, cols)
    for b in split_bands(rows, config.parts, halo):
        first = b.core_start - b.halo_above
        tile = image[first:b.core_start + b.core_rows + b.halo_below]
        tile = tile.clone() if _is_torch(tile) else np.ascontiguousarray(tile)
        out[b.core_start:b.core_start + b.core_rows] = adaptive_median_rows(
            tile, config.smax, b.halo_above, b.halo_above + b.core_rows, ctx=ctx)
    return out


# ---------------------------------------------------------------- W1 Wiener

@dataclass
class WindowStats:
    """reference WindowStats (proj/include/denoise/adaptive_median.hpp:16-22): uint8 planes."""
    zmin: object
    zmax: object
    zmed: object
    k: int = 0


def window_stats(image, k: int, ctx=None) -> WindowStats:
    """window_stats -- reference proj/src/adaptive_median.cpp:96-119: per-pixel min / median / max of the
    k x k window (edge replication), computed on the device (hyb_window_stats_u8)."""
    if k < 3 or k % 2 == 0:
        raise InvalidArgument(f"window size must be an odd integer >= 3, got {k}")
    rows, cols = _shape(image)
    outs = [_empty_like(image, rows, cols) for _ in range(3)]
    sp, spitch = capi.buf(image)
    ptrs = [capi.buf(o)[0] for o in outs]
    c = _ctx(ctx, image, *outs)
    check(lib.hyb_window_stats_u8(c, sp, spitch, rows, cols, k, ptrs[0], ptrs[1], ptrs[2], cols), c)
    return WindowStats(zmin=outs[0], zmax=outs[2], zmed=outs[1], k=k)


def wiener_local(f, win: int = 3, ctx=None):
    """W1 local-statistics Wiener on a whole image; returns (y, W) with W = sum of V."""
    rows, cols = _shape(f)
    y = _empty_like(f, rows, cols)
    fp, fpitch = capi.buf(f)
    yp, ypitch = capi.buf(y)
    w = ctypes.c_int64(0)
    c = _ctx(ctx, f, y)
    check(lib.hyb_wiener_u8(c, fp, fpitch, rows, cols, win, yp, ypitch, ctypes.byref(w)), c)
    return y, w.value


def noise_variance(noise_sum: int, pixel_count: int, win: int) -> float:
    """nu / 255^2 in the reference's [0, 1] intensity^2 units (HybridResult.sigma2)."""
    n = win * win
    return noise_sum / (n * n * pixel_count) / (255.0 * 255.0)


# ---------------------------------------------------------------- pipeline

@dataclass
class HybridResult:
    """HybridResult -- reference proj/include/denoise/pipeline.hpp:12-18 (+ the exact W)."""
    image: object
    sigma2: float
    t_adaptive: float
    t_wiener: float
    t_stretch: float
    noise_sum: int
    t_total: float


def hybrid_denoise(noisy, config: FilterConfig, reference=None, stretch_after_each: bool = False,
                   ctx=None) -> HybridResult:
    """hybrid_denoise -- reference proj/include/denoise/pipeline.hpp:25-27 (proj/src/pipeline.cpp:23-57)
    with the north_star's W1 Wiener in the stage-2 slot: the AMF (config.parts strips, bit-identical for
    every parts; config.gpus / device_ids devices), [contrast stretch when stretch_after_each], W1 with the
    noise of config.estimate_mode (REFERENCE needs `reference`, a float64 image in [0, 1] or a uint8
    image), [final contrast stretch when config.final_stretch]."""
    validate_config(config)
    rows, cols = _shape(noisy)
    if config.estimate_mode == EstimateMode.REFERENCE and reference is None:
        raise InvalidArgument("reference mode requires a reference image")
    if reference is not None and _shape(reference) != (rows, cols):
        raise InvalidArgument("reference image dimensions do not match")
    y = _empty_like(noisy, rows, cols)
    gp, gpitch = capi.buf(noisy)
    yp, ypitch = capi.buf(y)
    c = _config_ctx(ctx, config, noisy, y)
    if config.estimate_mode != EstimateMode.REFERENCE and not stretch_after_each:
        st = capi.HybStats()
        check(lib.hyb_hybrid_u8(c, gp, gpitch, rows, cols, config.smax, config.wiener_window, config.parts,
                                yp, ypitch, ctypes.byref(st)), c)
        res = HybridResult(y, st.sigma2, st.t_adaptive, st.t_wiener, 0.0, st.noise_sum, st.t_total)
    else:
        import time
        t0 = time.perf_counter()
        f = _empty_like(noisy, rows, cols)
        fp, fpitch = capi.buf(f)
        check(lib.hyb_amf_u8(c, gp, gpitch, rows, cols, 0, rows, config.smax, fp, fpitch, None, cols), c)
        t1 = time.perf_counter()
        t_stretch = 0.0
        if stretch_after_each:  # proj/src/pipeline.cpp:39-43 (uint8 stretch, rounded half up)
            check(lib.hyb_contrast_stretch_u8(c, fp, fpitch, rows, cols, fp, fpitch), c)
            t_stretch += time.perf_counter() - t1
        t2 = time.perf_counter()
        win = config.wiener_window
        n = win * win
        if config.estimate_mode == EstimateMode.REFERENCE:
            # sigma2 = mean((f - reference)^2) in [0, 1] units (proj/src/wiener.cpp:31-42), fed to the W1 gain as
            # W / (n^2 P) with P scaled by 64 (the rounding of W costs < 2^-6 / (n^2 P))
            fa = (f.cpu().numpy() if _is_torch(f) else f).astype(np.float64) / 255.0
            rn = reference.cpu().numpy() if _is_torch(reference) else np.asarray(reference)
            ra = rn.astype(np.float64) / 255.0 if rn.dtype == np.uint8 else rn.astype(np.float64)
            sigma2 = float(np.mean((fa - ra) ** 2))
            pn = rows * cols * 64
            w = int(np.floor(sigma2 * 255.0 * 255.0 * n * n * pn + 0.5))  # llround, as the C++ host
            wsum = 0
        else:
            wv = ctypes.c_int64(0)
            check(lib.hyb_wiener_stats_u8(c, fp, fpitch, rows, cols, 0, rows, win, ctypes.byref(wv)), c)
            w, pn = wv.value, rows * cols
            sigma2 = noise_variance(w, pn, win)
            wsum = w
        wv = ctypes.c_int64(w)
        check(lib.hyb_wiener_gain_u8(c, fp, fpitch, rows, cols, 0, rows, win, ctypes.byref(wv), pn, yp, ypitch), c)
        res = HybridResult(y, sigma2, t1 - t0, time.perf_counter() - t2, t_stretch, wsum, time.perf_counter() - t0)
    if config.final_stretch:  # proj/src/pipeline.cpp:55-57
        import time
        t3 = time.perf_counter()
        check(lib.hyb_contrast_stretch_u8(c, yp, ypitch, rows, cols, yp, ypitch), c)
        res.t_stretch += time.perf_counter() - t3
    return res


def contrast_stretch(image, ctx=None):
    """contrast_stretch -- reference proj/src/pipeline.cpp:10-21.  float64 images: the reference's own
    (p - lo) / (hi - lo) (bit-identical); uint8 images: that quotient scaled to 0..255, rounded half up
    (lo -> 0, hi -> 255).  Constant images are returned unchanged."""
    is_f64 = (str(image.dtype) == "torch.float64") if _is_torch(image) else np.asarray(image).dtype == np.float64
    if is_f64:
        p, pitch, rows, cols = _f64(image)
        if _is_torch(image):
            import torch
            out = torch.empty((rows, cols), dtype=torch.float64, device=image.device)
            op = out.data_ptr()
        else:
            out = np.empty((rows, cols), np.float64)
            op = out.ctypes.data
        c = _ctx(ctx, image, out)
        check(lib.hyb_contrast_stretch_f64(c, p, pitch, rows, cols, op, cols), c)
        return out
    rows, cols = _shape(image)
    out = _empty_like(image, rows, cols)
    sp, spitch = capi.buf(image)
    dp, dpitch = capi.buf(out)
    c = _ctx(ctx, image, out)
    check(lib.hyb_contrast_stretch_u8(c, sp, spitch, rows, cols, dp, dpitch), c)
    return out


def hybrid_denoise_stretched(noisy, config: FilterConfig, ctx=None) -> HybridResult:
    """hybrid_denoise stages 1-3 (reference proj/src/pipeline.cpp:23-57, stretch_after_each = false):
    AMF, W1, then the final contrast_stretch."""
    validate_config(config)
    rows, cols = _shape(noisy)
    y = _empty_like(noisy, rows, cols)
    gp, gpitch = capi.buf(noisy)
    yp, ypitch = capi.buf(y)
    st = capi.HybStats()
    c = _config_ctx(ctx, config, noisy, y)
    check(lib.hyb_hybrid_stretch_u8(c, gp, gpitch, rows, cols, config.smax, config.wiener_window, config.parts,
                                    yp, ypitch, ctypes.byref(st)), c)
    return HybridResult(y, st.sigma2, st.t_adaptive, st.t_wiener, 0.0, st.noise_sum, st.t_total)


def hybrid_denoise_batch(stack, smax: int, win: int, ctx=None):
    """CT-stack hybrid: each slice filtered independently (own noise estimate).  Returns
    (filtered stack, per-slice W)."""
    if stack.ndim != 3:
        raise InvalidArgument("expected a (slices, rows, cols) stack")
    n, rows, cols = (int(s) for s in stack.shape)
    if _is_torch(stack):
        import torch
        y = torch.empty_like(stack)
        sstride = stack.stride(0)
        ystride = y.stride(0)
    else:
        stack = np.ascontiguousarray(stack)
        y = np.empty_like(stack)
        sstride, ystride = stack.strides[0], y.strides[0]
    gp, gpitch = capi.buf(stack)
    yp, ypitch = capi.buf(y)
    w = (ctypes.c_int64 * n)()
    c = _ctx(ctx, stack, y)
    check(lib.hyb_hybrid_batch_u8(c, gp, gpitch, sstride, n, rows, cols, smax, win, yp, ypitch, ystride, w), c)
    return y, list(w)


# ---------------------------------------------------------------- uint8 <-> reference doubles

def to_u8(img: np.ndarray) -> np.ndarray:
    """Reference Image doubles -> uint8 with lround(p * 255) (proj/src/pgm_io.cpp:115); rejects
    off-grid values, which have no exact uint8 representation."""
    q = np.clip(np.floor(np.asarray(img, np.float64) * 255.0 + 0.5), 0, 255)
    if not np.array_equal(q / 255.0, img):
        raise InvalidArgument("image has values off the k/255 grid; no exact uint8 representation")
    return q.astype(np.uint8)


def to_unit(img_u8) -> np.ndarray:
    """uint8 -> the reference's [0, 1] doubles, k/255 (proj/src/pgm_io.cpp:73,88)."""
    return np.asarray(img_u8, np.float64) / 255.0


# ---------------------------------------------------------------- PGM I/O

def _pgm_error(path, what):
    raise RuntimeError(f"pgm {path}: {what}")


def load_pgm(path):
    """load_pgm -- reference proj/src/pgm_io.cpp:49-103: P5 or P2, maxval 1..65535.  maxval 255 files
    return the uint8 raster (exactly the reference's k/255 doubles, ready for the uint8 path); other
    maxvals return float64 samples / maxval like the reference.  Errors are RuntimeError("pgm <path>:
    ...") with the reference's texts."""
    try:
        data = open(path, "rb").read()
    except OSError:
        _pgm_error(path, "cannot open file")
    if len(data) < 2 or data[0:1] != b"P" or data[1:2] not in (b"2", b"5"):
        magic = data[:2].decode("latin-1") if len(data) >= 2 else ""
        _pgm_error(path, f'unsupported magic "{magic}" (want P2 or P5)')
    binary = data[1:2] == b"5"
    i = 2

    def skip(i):
        while i < len(data):
            c = data[i:i + 1]
            if c == b"#":
                while i < len(data) and data[i:i + 1] != b"\n":
                    i += 1
            elif c.isspace():
                i += 1
            else:
                break
        return i

    def number(i):
        j = i
        while j < len(data) and data[j:j + 1].isdigit():
            j += 1
        return (int(data[i:j]) if j > i else None), j

    fields = []
    for name in ("width", "height", "maxval"):
        i = skip(i)
        v, i = number(i)
        if v is None:
            _pgm_error(path, f"malformed header: missing {name}")
        if v > 1000000000:
            _pgm_error(path, f"header field out of range: {name}")
        fields.append(v)
    cols, rows, maxval = fields
    if cols < 1 or rows < 1:
        _pgm_error(path, "non-positive dimensions in header")
    if maxval < 1 or maxval > 65535:
        _pgm_error(path, f"maxval {maxval} out of range [1, 65535]")
    count = rows * cols
    if binary:
        if i >= len(data) or not data[i:i + 1].isspace():
            _pgm_error(path, "missing separator before pixel data")
        i += 1
        bps = 2 if maxval > 255 else 1
        if len(data) - i < count * bps:
            _pgm_error(path, "truncated pixel data")
        raw = np.frombuffer(data, dtype=">u2" if bps == 2 else np.uint8, count=count, offset=i).astype(np.int64)
    else:
        vals = []
        for k in range(count):
            i = skip(i)
            v, i = number(i)
            if v is None:
                _pgm_error(path, f"truncated pixel data at sample {k}")
            vals.append(v)
        raw = np.array(vals, dtype=np.int64)
    bad = raw > maxval
    if bad.any():
        _pgm_error(path, f"sample {int(raw[np.argmax(bad)])} exceeds maxval")
    raw = raw.reshape(rows, cols)
    return raw.astype(np.uint8) if maxval == 255 else raw / float(maxval)


def save_pgm(image, path):
    """save_pgm -- reference proj/src/pgm_io.cpp:105-120: P5, maxval 255.  uint8 images are written as
    is; float images in [0, 1] are quantised round(p * 255) with halves away from zero, clipped."""
    img = np.asarray(image.cpu() if _is_torch(image) else image)
    if img.dtype == np.uint8:
        raw = img
    else:
        x = img.astype(np.float64) * 255.0
        raw = np.clip(np.where(x >= 0, np.floor(x + 0.5), np.ceil(x - 0.5)), 0, 255).astype(np.uint8)
    rows, cols = raw.shape
    try:
        with open(path, "wb") as f:
            f.write(f"P5\n{cols} {rows}\n255\n".encode())
            f.write(np.ascontiguousarray(raw).tobytes())
    except OSError:
        _pgm_error(path, "cannot open file for writing")


# ---------------------------------------------------------------- the reference's Wiener stage (8(f) row 3)

def _f64(img):
    """(pointer, pitch in elements, rows, cols) of a float64 numpy array / torch tensor (2-D)."""
    if _is_torch(img):
        import torch
        if img.dtype != torch.float64 or img.dim() != 2 or img.stride(1) != 1:
            raise InvalidArgument("expected a 2-D float64 tensor with unit column stride")
        return img.data_ptr(), img.stride(0), int(img.shape[0]), int(img.shape[1])
    a = np.asarray(img)
    if a.dtype != np.float64 or a.ndim != 2 or a.strides[1] != 8:
        raise InvalidArgument("expected a 2-D float64 array with unit column stride")
    return a.ctypes.data, a.strides[0] // 8, a.shape[0], a.shape[1]


def wiener_filter(image, sigma2: float, clamp: bool = True, ctx=None):
    """wiener_filter -- reference proj/src/wiener.cpp:54-77: frequency-domain Wiener on a float64
    image (per-bin gain (P - N0) / P, N0 = rows * cols * sigma2), clamped to [0, 1] by default."""
    p, pitch, rows, cols = _f64(image)
    if _is_torch(image):
        import torch
        out = torch.empty((rows, cols), dtype=torch.float64, device=image.device)
        op, opitch = out.data_ptr(), cols
    else:
        out = np.empty((rows, cols), np.float64)
        op, opitch = out.ctypes.data, cols
    c = _ctx(ctx, image, out)
    check(lib.hyb_wiener_freq_f64(c, p, pitch, rows, cols, float(sigma2), int(bool(clamp)), op, opitch), c)
    return out


def estimate_noise_variance(image, reference=None, ctx=None):
    """estimate_noise_variance -- reference proj/src/wiener.cpp:30-52 on float64 images: with a reference
    the mean squared difference, else (median |p - median3(p)| / 0.6745)^2.  Returns (sigma2, source)."""
    p, pitch, rows, cols = _f64(image)
    c = _ctx(ctx, image, reference)
    out = ctypes.c_double(0.0)
    if reference is not None:
        rp, rpitch, rr, rc = _f64(reference)
        if (rr, rc) != (rows, cols):
            raise InvalidArgument("reference image dimensions do not match")
        check(lib.hyb_noise_reference_f64(c, p, pitch, rp, rpitch, rows, cols, ctypes.byref(out)), c)
        return out.value, "reference"
    check(lib.hyb_noise_robust_f64(c, p, pitch, rows, cols, ctypes.byref(out)), c)
    return out.value, "robust"


def hybrid_denoise_reference(noisy, config: FilterConfig, reference=None, stretch_after_each: bool = False,
                             ctx=None) -> HybridResult:
    """The reference's full hybrid_denoise (proj/src/pipeline.cpp:23-57) on the GPU: adaptive median
    (bands per config), [contrast stretch], noise estimate (robust, or the mean squared difference to
    `reference`), frequency-domain Wiener (clamped), final contrast stretch.  noisy: uint8 (k/255);
    reference: float64 in [0, 1] or None.  The image is float64 like the reference's."""
    import time
    validate_config(config)
    rows, cols = _shape(noisy)
    if reference is not None and _shape(reference) != (rows, cols):
        raise InvalidArgument("reference image dimensions do not match")
    t0 = time.perf_counter()
    f = adaptive_median_parallel(noisy, config, ctx=ctx)
    f = (f.double() / 255.0) if _is_torch(f) else np.asarray(f, np.float64) / 255.0
    t1 = time.perf_counter()
    t_stretch = 0.0
    if stretch_after_each:
        f = contrast_stretch(f, ctx=ctx)
        t_stretch += time.perf_counter() - t1
    t2 = time.perf_counter()
    sigma2, _ = estimate_noise_variance(f, reference, ctx=ctx)
    y = wiener_filter(f, sigma2, clamp=True, ctx=ctx)
    t3 = time.perf_counter()
    y = contrast_stretch(y, ctx=ctx)
    t_stretch += time.perf_counter() - t3
    return HybridResult(y, sigma2, t1 - t0, t3 - t2, t_stretch, 0, time.perf_counter() - t0)

