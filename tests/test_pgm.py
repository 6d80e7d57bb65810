"""PGM I/O, CPU only: the C++ host driver's load_pgm / save_pgm against the
reference's cases (tests/cpp/test_pgm.cpp), and the Python mirror (denoise.load_pgm / save_pgm) on
the same cases plus cross-reading files written by the other side."""
import os
import subprocess

import numpy as np
import pytest

from paper_2005_05371_b200 import denoise

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_pgm_io():
    exe = os.path.join(ROOT, "tests", "cpp", "test_pgm")
    assert os.path.exists(exe), "build with `make`"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr


def _write(path, data: bytes):
    with open(path, "wb") as f:
        f.write(data)


def test_python_pgm_reference_cases(tmp_path):
    p = tmp_path / "p5.pgm"
    _write(p, b"P5\n2 2\n255\n\x00\x80\xff\x40")
    img = denoise.load_pgm(p)
    assert img.dtype == np.uint8 and img.tolist() == [[0, 128], [255, 64]]
    _write(p, b"P2 1 1 255 255")
    assert denoise.load_pgm(p).tolist() == [[255]]
    _write(p, b"P5\n# a comment\n1 1\n65535\n\xff\xff")
    v = denoise.load_pgm(p)
    assert v.dtype == np.float64 and v[0, 0] == 1.0  # maxval != 255: samples / maxval (reference doubles)
    _write(p, b"P6\n1 1\n255\n\x01\x02\x03")
    with pytest.raises(RuntimeError, match="unsupported magic"):
        denoise.load_pgm(p)
    _write(p, b"P5\n2 2\n255\n\x00\x80")
    with pytest.raises(RuntimeError, match="truncated"):
        denoise.load_pgm(p)
    _write(p, b"P2 2 1 10 3 11")
    with pytest.raises(RuntimeError, match="exceeds maxval"):
        denoise.load_pgm(p)


def test_python_pgm_writer_and_round_trip(tmp_path):
    p = tmp_path / "w.pgm"
    denoise.save_pgm(np.array([[0, 255]], np.uint8), p)
    assert open(p, "rb").read() == b"P5\n2 1\n255\n\x00\xff"
    denoise.save_pgm(np.array([[0.5]]), p)  # doubles: round half away from zero, 127.5 -> 128
    assert denoise.load_pgm(p).tolist() == [[128]]
    grid = np.arange(256, dtype=np.uint8).reshape(16, 16)
    denoise.save_pgm(grid, p)
    np.testing.assert_array_equal(denoise.load_pgm(p), grid)
    rng = np.random.default_rng(99)
    img = rng.random((64, 64))
    denoise.save_pgm(img, p)
    assert np.max(np.abs(denoise.load_pgm(p) / 255.0 - img)) <= 1 / 510 + 1e-12
