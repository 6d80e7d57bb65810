"""CPU checker for the hybrid AMF + W1 Wiener path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs may
import this package, and only as the checker or the CPU baseline, never as the product path.

* ``liboracle.so`` (hyb_oracle.c): C restatement of detail::adaptive_median_rows (reference
  proj/src/adaptive_median.cpp:123-215) on uint8 and of the W1 local Wiener (
  no reference implementation exists -> W1 parity is "unpinned" w.r.t. the reference).
* ``_ref/libref.so``: the UNMODIFIED reference sources compiled from /root/reference by
  oracle/Makefile plus ref_shim.cpp.  Pins the AMF restatement and serves as the CPU baseline.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int64, c_size_t, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref.so")


def _load_oracle():
    lib = ctypes.CDLL(ORACLE_SO)
    P = c_void_p
    lib.hyb_oracle_amf_u8.argtypes = [P, c_size_t, c_int, c_int, c_int, c_int, c_int, P, c_size_t, P, c_size_t]
    lib.hyb_oracle_wiener_stats_u8.argtypes = [P, c_size_t, c_int, c_int, c_int, c_int, c_int, POINTER(c_int64)]
    lib.hyb_oracle_wiener_gain_u8.argtypes = [P, c_size_t, c_int, c_int, c_int, c_int, c_int, c_int64, c_int64,
                                              P, c_size_t]
    lib.hyb_oracle_hybrid_u8.argtypes = [P, c_size_t, c_int, c_int, c_int, c_int, P, P, c_size_t, POINTER(c_int64)]
    lib.hyb_oracle_validate_smax.argtypes = [c_int]
    lib.hyb_oracle_window_stats_u8.argtypes = [P, c_size_t, c_int, c_int, c_int, P, P, P, c_size_t]
    lib.hyb_oracle_contrast_stretch_u8.argtypes = [P, c_size_t, c_int, c_int, P, c_size_t]
    lib.oracle_make_phantom_u8.argtypes = [c_int, c_int, c_int, c_double, c_double, c_uint64, P, c_size_t]
    return lib


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            raise ImportError(f"{ORACLE_SO} missing: run `make -C oracle`")
        _lib = _load_oracle()
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference itself (compiled in oracle/_ref)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise ImportError(f"{REF_SO} missing: run `make -C oracle` where /root/reference exists")
        r = ctypes.CDLL(REF_SO)
        P = c_void_p
        r.ref_last_error.restype = ctypes.c_char_p
        r.ref_validate_smax.argtypes = [c_int]
        r.ref_amf_rows_u8.argtypes = [P, c_size_t, c_int, c_int, c_int, c_int, c_int, P, c_size_t, P, c_size_t]
        r.ref_amf_parallel_u8.argtypes = [P, c_size_t, c_int, c_int, c_int, c_int, c_int, c_int, P, c_size_t,
                                          POINTER(c_double)]
        r.ref_window_stats_u8.argtypes = [P, c_size_t, c_int, c_int, c_int, P, P, P, c_size_t]
        r.ref_split_bands.argtypes = [c_int, c_int, c_int, c_int, POINTER(c_int)]
        r.ref_rng_uniform.argtypes = [c_uint64, c_int, POINTER(c_double)]
        r.ref_rng_normal.argtypes = [c_uint64, c_int, POINTER(c_double)]
        r.ref_salt_pepper_count.argtypes = [c_int, c_int, c_double, c_double, c_uint64]
        r.ref_rng_u64.argtypes = [c_uint64, c_int, POINTER(c_uint64)]
        r.ref_random_image_u8.argtypes = [c_int, c_int, c_uint64, c_double, c_uint64, P]
        r.ref_noisy_phantom_u8.argtypes = [c_int, c_int, c_uint64, P]
        r.ref_hybrid_baseline.argtypes = [P, c_int, c_int, c_int, c_int, c_int, P, POINTER(c_double),
                                          POINTER(c_double)]
        _ref = r
    return _ref


def _u8(a):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return a, a.ctypes.data


# ---------------- oracle (C restatement) ----------------

def amf(img, smax, row_begin=0, row_end=None, finalized_at=False):
    img, p = _u8(img)
    rows, cols = img.shape
    row_end = rows if row_end is None else row_end
    out = np.empty((max(row_end - row_begin, 0), cols), np.uint8)
    fin = np.empty_like(out) if finalized_at else None
    st = lib().hyb_oracle_amf_u8(p, cols, rows, cols, row_begin, row_end, smax, out.ctypes.data, cols,
                                 fin.ctypes.data if fin is not None else None, cols)
    if st:
        raise ValueError(f"oracle amf rejected smax={smax} range=[{row_begin},{row_end}) of {rows}")
    return (out, fin) if finalized_at else out


def window_stats(img, k):
    """(zmin, zmed, zmax) planes of the k x k windows (reference window_stats,
    proj/src/adaptive_median.cpp:96-119)."""
    img, p = _u8(img)
    rows, cols = img.shape
    out = [np.empty((rows, cols), np.uint8) for _ in range(3)]
    st = lib().hyb_oracle_window_stats_u8(p, cols, rows, cols, k, *(o.ctypes.data for o in out), cols)
    if st:
        raise ValueError(f"window size must be an odd integer >= 3, got {k}")
    return tuple(out)


def ref_window_stats(img, k):
    """The reference's own window_stats on k/255 doubles, mapped back to uint8."""
    img, p = _u8(img)
    rows, cols = img.shape
    out = [np.empty((rows, cols), np.uint8) for _ in range(3)]
    if ref().ref_window_stats_u8(p, cols, rows, cols, k, *(o.ctypes.data for o in out), cols):
        raise ValueError(ref().ref_last_error().decode())
    return tuple(out)


def wiener_stats(f, win, row_begin=0, row_end=None):
    f, p = _u8(f)
    rows, cols = f.shape
    row_end = rows if row_end is None else row_end
    w = c_int64(0)
    st = lib().hyb_oracle_wiener_stats_u8(p, cols, rows, cols, row_begin, row_end, win, ctypes.byref(w))
    if st:
        raise ValueError("oracle wiener_stats rejected its arguments")
    return w.value


def wiener_gain(f, win, noise_sum, pixel_count, row_begin=0, row_end=None):
    f, p = _u8(f)
    rows, cols = f.shape
    row_end = rows if row_end is None else row_end
    y = np.empty((row_end - row_begin, cols), np.uint8)
    st = lib().hyb_oracle_wiener_gain_u8(p, cols, rows, cols, row_begin, row_end, win, noise_sum, pixel_count,
                                         y.ctypes.data, cols)
    if st:
        raise ValueError("oracle wiener_gain rejected its arguments")
    return y


def wiener(f, win):
    w = wiener_stats(f, win)
    return wiener_gain(f, win, w, f.shape[0] * f.shape[1]), w


def hybrid(g, smax, win):
    g, p = _u8(g)
    rows, cols = g.shape
    work = np.empty_like(g)
    y = np.empty_like(g)
    w = c_int64(0)
    st = lib().hyb_oracle_hybrid_u8(p, cols, rows, cols, smax, win, work.ctypes.data, y.ctypes.data, cols,
                                    ctypes.byref(w))
    if st:
        raise ValueError("oracle hybrid rejected its arguments")
    return y, w.value


def make_phantom(rows, cols, n_ellipses, sigma, density, seed):
    """The BASELINE.json phantom (the product's phantom.cpp compiled into liboracle.so): identical bytes
    to paper_2005_05371_b200.capi.make_phantom, for the CPU reference arm (which must not load the
    product library)."""
    out = np.empty((rows, cols), np.uint8)
    if lib().oracle_make_phantom_u8(rows, cols, n_ellipses, float(sigma), float(density), seed, out.ctypes.data,
                                    cols):
        raise ValueError("bad phantom parameters")
    return out


def _bands(rows, threads):
    threads = max(1, min(threads, rows))
    return [(rows * i // threads, rows * (i + 1) // threads) for i in range(threads)]


def _pool_map(fn, items, threads):
    # ctypes releases the GIL for the foreign call, so row bands run in parallel
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, threads)) as ex:
        return list(ex.map(fn, items))


def amf_threaded(img, smax, threads=None):
    """amf() of the whole image, row bands in parallel (each band's windows read the whole source)."""
    img, _ = _u8(img)
    threads = threads or os.cpu_count() or 1
    parts = _pool_map(lambda ab: amf(img, smax, ab[0], ab[1]), _bands(img.shape[0], threads), threads)
    return np.concatenate(parts, axis=0)


def wiener_threaded(f, win, threads=None):
    """wiener() with the statistics and the gain over row bands in parallel (W is an exact int64 sum)."""
    f, _ = _u8(f)
    threads = threads or os.cpu_count() or 1
    bands = _bands(f.shape[0], threads)
    w = sum(_pool_map(lambda ab: wiener_stats(f, win, ab[0], ab[1]), bands, threads))
    P = f.shape[0] * f.shape[1]
    y = np.concatenate(_pool_map(lambda ab: wiener_gain(f, win, w, P, ab[0], ab[1]), bands, threads), axis=0)
    return y, w


def hybrid_threaded(g, smax, win, threads=None):
    f = amf_threaded(g, smax, threads)
    return wiener_threaded(f, win, threads)


def hybrid_many(images, smax, win, threads=None):
    """oracle hybrid() of independent images (a CT stack), one image per worker thread."""
    threads = threads or os.cpu_count() or 1
    return _pool_map(lambda g: hybrid(g, smax, win), list(images), threads)


# ---------------- the reference itself (oracle/_ref) ----------------

def ref_amf_rows(img, smax, row_begin=0, row_end=None, finalized_at=False):
    img, p = _u8(img)
    rows, cols = img.shape
    row_end = rows if row_end is None else row_end
    out = np.empty((max(row_end - row_begin, 0), cols), np.uint8)
    fin = np.empty_like(out) if finalized_at else None
    st = ref().ref_amf_rows_u8(p, cols, rows, cols, row_begin, row_end, smax, out.ctypes.data, cols,
                               fin.ctypes.data if fin is not None else None, cols)
    if st:
        raise ValueError(ref().ref_last_error().decode())
    return (out, fin) if finalized_at else out


def ref_amf_parallel(img, smax, parts, workers, use_halo=True):
    img, p = _u8(img)
    rows, cols = img.shape
    out = np.empty_like(img)
    sec = c_double(0)
    st = ref().ref_amf_parallel_u8(p, cols, rows, cols, smax, parts, workers, int(use_halo), out.ctypes.data,
                                   cols, ctypes.byref(sec))
    if st:
        raise ValueError(ref().ref_last_error().decode())
    return out, sec.value


def ref_split_bands(rows, cols, parts, halo):
    out = (c_int * (4 * parts))()
    st = ref().ref_split_bands(rows, cols, parts, halo, out)
    if st:
        raise ValueError(ref().ref_last_error().decode())
    return [tuple(out[4 * i:4 * i + 4]) for i in range(parts)]


def ref_rng(seed, n, normal=False):
    out = (c_double * n)()
    (ref().ref_rng_normal if normal else ref().ref_rng_uniform)(seed, n, out)
    return np.frombuffer(out, dtype=np.float64).copy()


def ref_rng_u64(seed, n):
    out = (c_uint64 * n)()
    ref().ref_rng_u64(seed, n, out)
    return [int(v) for v in out]


def ref_random_image(rows, cols, seed, density=0.0, sp_seed=0):
    out = np.empty((rows, cols), np.uint8)
    if ref().ref_random_image_u8(rows, cols, seed, density, sp_seed, out.ctypes.data):
        raise ValueError(ref().ref_last_error().decode())
    return out


def ref_noisy_phantom(rows, cols, seed):
    out = np.empty((rows, cols), np.uint8)
    if ref().ref_noisy_phantom_u8(rows, cols, seed, out.ctypes.data):
        raise ValueError(ref().ref_last_error().decode())
    return out


def ref_hybrid_baseline(g, smax, win, threads):
    """Reference AMF (adaptive_median_parallel, parts = workers = threads) + W1 oracle on threads."""
    g, p = _u8(g)
    rows, cols = g.shape
    y = np.empty_like(g)
    ta, tw = c_double(0), c_double(0)
    st = ref().ref_hybrid_baseline(p, rows, cols, smax, win, threads, y.ctypes.data, ctypes.byref(ta),
                                   ctypes.byref(tw))
    if st:
        raise ValueError(ref().ref_last_error().decode())
    return y, ta.value, tw.value


def contrast_stretch(img):
    """uint8 contrast stretch (proj/src/pipeline.cpp:10-21 restated, rounded half up to 0..255)."""
    img, p = _u8(img)
    rows, cols = img.shape
    out = np.empty_like(img)
    if lib().hyb_oracle_contrast_stretch_u8(p, cols, rows, cols, out.ctypes.data, cols):
        raise ValueError("oracle contrast_stretch rejected its arguments")
    return out


# -------- the reference's Wiener stage, restated in numpy (proj/src/wiener.cpp:30-77, dft2.cpp:32-56)

def wiener_freq(img, sigma2, clamp=True):
    """wiener_filter via numpy's double FFT (the reference uses FFTW, double)."""
    x = np.asarray(img, np.float64)
    if sigma2 == 0.0:
        return np.clip(x, 0.0, 1.0) if clamp else x.copy()
    spec = np.fft.fft2(x)
    p = spec.real ** 2 + spec.imag ** 2
    n0 = x.shape[0] * x.shape[1] * sigma2
    g = np.where(p > n0, (p - n0) / np.where(p > 0, p, 1.0), 0.0)
    out = np.fft.ifft2(spec * g).real
    return np.clip(out, 0.0, 1.0) if clamp else out


def wiener_direct(img, sigma2):
    """wiener_filter by direct-summation DFT (matrix form), like the reference's test oracle."""
    x = np.asarray(img, np.float64)
    m, n = x.shape
    wm = np.exp(-2j * np.pi * np.outer(np.arange(m), np.arange(m)) / m)
    wn = np.exp(-2j * np.pi * np.outer(np.arange(n), np.arange(n)) / n)
    spec = wm @ x @ wn
    p = np.abs(spec) ** 2
    n0 = m * n * sigma2
    g = np.where(p > n0, (p - n0) / np.where(p > 0, p, 1.0), 0.0)
    return (np.conj(wm) @ (spec * g) @ np.conj(wn)).real / (m * n)


def noise_robust(img):
    """(median |p - median3(p)| / 0.6745)^2, median3 with replicated borders, even counts averaged."""
    x = np.asarray(img, np.float64)
    pad = np.pad(x, 1, mode="edge")
    win = np.stack([pad[dr:dr + x.shape[0], dc:dc + x.shape[1]] for dr in range(3) for dc in range(3)])
    med3 = np.median(win, axis=0)
    sigma = np.median(np.abs(x - med3)) / 0.6745
    return sigma * sigma


def noise_reference(a, b):
    d = np.asarray(a, np.float64) - np.asarray(b, np.float64)
    return float(np.mean(d * d))


def contrast_stretch_f64(img):
    """proj/src/pipeline.cpp:10-21 verbatim in float64."""
    x = np.asarray(img, np.float64)
    lo, hi = x.min(), x.max()
    return x.copy() if hi == lo else (x - lo) / (hi - lo)


def hybrid_reference(g, smax, reference=None, stretch_after_each=False):
    """The reference's full hybrid_denoise chain restated: AMF (C oracle), [stretch], estimate, frequency
    Wiener (numpy FFT), final stretch."""
    f = amf(g, smax).astype(np.float64) / 255.0
    if stretch_after_each:
        f = contrast_stretch_f64(f)
    sigma2 = noise_reference(f, reference) if reference is not None else noise_robust(f)
    return contrast_stretch_f64(wiener_freq(f, sigma2, True)), sigma2

