"""CPU: libhybrid_cuda.so loads and exports every symbol include/hybrid_cuda.h declares; host-only
entry points work without a GPU and no compute entry point silently runs on the CPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2005_05371_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "hybrid_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hyb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    names = header_functions()
    assert len(names) >= 15
    lib = ctypes.CDLL(capi.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(capi.EXPORTED)


def test_library_is_sm100a():
    blob = open(capi.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob or b"sm_100" in blob


def test_validate_entry_points():
    assert capi.lib.hyb_validate_smax(3) == capi.HYB_OK
    assert capi.lib.hyb_validate_smax(11) == capi.HYB_OK
    for bad in (4, 1, 0, -3):
        assert capi.lib.hyb_validate_smax(bad) == capi.HYB_EINVAL
    assert capi.lib.hyb_validate_config(11, 4, 4) == capi.HYB_OK
    assert capi.lib.hyb_validate_config(4, 1, 1) == capi.HYB_EINVAL
    assert capi.lib.hyb_validate_config(3, 0, 1) == capi.HYB_EINVAL
    assert capi.lib.hyb_validate_config(3, 1, 0) == capi.HYB_EINVAL


def test_phantom_generator_is_deterministic():
    a = capi.make_phantom(64, 80, 5, 10.0, 0.1, 3)
    b = capi.make_phantom(64, 80, 5, 10.0, 0.1, 3)
    c = capi.make_phantom(64, 80, 5, 10.0, 0.1, 4)
    np.testing.assert_array_equal(a, b)
    assert (a != c).any()
    with pytest.raises(capi.InvalidArgument):
        capi.make_phantom(0, 5, 1, 1.0, 0.1, 0)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    st = ctypes.c_int(0)
    ctx = capi.lib.hyb_create(0, ctypes.byref(st))
    assert not ctx and st.value == capi.HYB_ECUDA
    with pytest.raises(capi.CudaError):
        capi.Context(0)
