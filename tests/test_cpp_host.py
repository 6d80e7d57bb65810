"""GPU: runs the C++ host-driver test binary (tests/cpp/test_host.cpp), the reference's hot-path
unit tests re-expressed against denoise_cuda:: with the C oracle as the checker."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_host_driver():
    exe = os.path.join(ROOT, "tests", "cpp", "test_host")
    assert os.path.exists(exe), "build with `make`"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
