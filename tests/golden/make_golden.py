#!/usr/bin/env python3
"""Regenerates the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

The reference's own sources are compiled here into oracle/_ref/libref.so (oracle/Makefile, from
/root/reference, never copied).  This script re-runs the reference's AMF test fixtures on the
uint8 grid (k/255 doubles, exact for the AMF; SURVEY.md finding 4) and stores inputs + reference
outputs, so the GPU tests (which run where /root/reference does not exist) compare against the
reference's results.  The W1 Wiener has no reference implementation: wiener_kat.json holds
hand-checkable cases computed here with exact rational arithmetic (fractions.Fraction),
independently of the C oracle.

    python tests/golden/make_golden.py               (every fixture)
    python tests/golden/make_golden.py window_stats  (window_stats_reference.npz only)
"""
import json
import os
import sys
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402


def amf_case(img, smax):
    out, fin = oracle.ref_amf_rows(img, smax, finalized_at=True)
    return out, fin


def build_amf():
    cases = {}

    def add(name, img, smaxes, **meta):
        cases[f"{name}/input"] = img
        for s in smaxes:
            out, fin = amf_case(img, s)
            cases[f"{name}/out_s{s}"] = out
            cases[f"{name}/fin_s{s}"] = fin

    # KATs, rank-compressed (proj/tests/test_adaptive_median.cpp:26-38, :61-78)
    add("kat_ramp3", np.arange(1, 10, dtype=np.uint8).reshape(3, 3), [3])
    grad = np.fromfunction(lambda r, c: r + c + 1, (5, 5)).astype(np.uint8)
    grad[2, 2] = 255
    add("kat_gradient_salt", grad, [3])
    add("kat_constant", np.full((9, 9), 178, np.uint8), [11])

    # oracle equivalence, 40 trials (proj/tests/test_adaptive_median.cpp:80-96), quantised
    seed = 1000
    for trial in range(40):
        d = oracle.ref_rng_u64(seed, 2)
        rows, cols = 8 + d[0] % 25, 8 + d[1] % 25
        img = oracle.ref_random_image(rows, cols, seed + 1, 0.2 if trial % 2 == 0 else 0.0, seed + 2)
        add(f"unit40_{trial:02d}", img, [3, 5, 7, 11])
        seed += 10

    # acceptance criterion 2: 100 small images (proj/tests/acceptance.cpp:84-101)
    d = oracle.ref_rng_u64(777, 200)
    for trial in range(100):
        rows, cols = 1 + d[2 * trial] % 32, 1 + d[2 * trial + 1] % 32
        img = oracle.ref_random_image(rows, cols, 5000 + trial, 0.25 if trial % 3 == 0 else 0.0, 6000 + trial)
        add(f"oracle100_{trial:03d}", img, [3, 5, 7, 11])

    # acceptance criterion 1: 20 images 63..257 (proj/tests/acceptance.cpp:50-80)
    d = oracle.ref_rng_u64(2026, 40)
    for trial in range(20):
        rows, cols = 63 + d[2 * trial] % 195, 63 + d[2 * trial + 1] % 195
        if trial % 2 == 0:
            rows |= 1
        img = oracle.ref_random_image(rows, cols, 3000 + trial, 0.2 if trial % 2 == 1 else 0.0, 4000 + trial)
        add(f"exact20_{trial:02d}", img, [3, 7, 11])

    # parallel fixtures (proj/tests/test_parallel.cpp:20-24, :54-109)
    add("par_64x64_s3", oracle.ref_noisy_phantom(64, 64, 3), [3, 11])
    add("par_63x57_s4", oracle.ref_noisy_phantom(63, 57, 4), [7])
    add("par_48x32_s5", oracle.ref_noisy_phantom(48, 32, 5), [11])
    img = oracle.ref_noisy_phantom(40, 40, 6)
    add("par_40x40_s6", img, [11])
    bare, _ = oracle.ref_amf_parallel(img, 11, 4, 2, use_halo=False)
    cases["par_40x40_s6/nohalo_p4_s11"] = bare
    add("par_30x26_700", oracle.ref_random_image(30, 26, 700, 0.2, 701), [5])
    # finalized_at agreement across smax (proj/tests/test_adaptive_median.cpp:108-130)
    add("fin_20x20_70", oracle.ref_random_image(20, 20, 70, 0.25, 71), [5, 11])
    return cases


def wiener_exact(f, win):
    """Independent W1 restatement in exact rationals."""
    f = np.asarray(f, dtype=np.int64)
    rows, cols = f.shape
    rad = win // 2
    n = win * win
    S1 = np.zeros_like(f)
    S2 = np.zeros_like(f)
    for r in range(rows):
        for c in range(cols):
            a = b = 0
            for dr in range(-rad, rad + 1):
                for dc in range(-rad, rad + 1):
                    x = int(f[min(max(r + dr, 0), rows - 1), min(max(c + dc, 0), cols - 1)])
                    a += x
                    b += x * x
            S1[r, c], S2[r, c] = a, b
    V = n * S2 - S1 * S1
    W = int(V.sum())
    P = rows * cols
    nu = Fraction(W, n * n * P)
    y = np.zeros((rows, cols), dtype=np.int64)
    for r in range(rows):
        for c in range(cols):
            mu = Fraction(int(S1[r, c]), n)
            v = Fraction(int(V[r, c]), n * n)
            if v <= nu:
                val = mu
            else:
                val = mu + (v - nu) / v * (int(f[r, c]) - mu)
            q = (val + Fraction(1, 2)).__floor__()  # round half away from zero (val >= 0)
            y[r, c] = min(max(q, 0), 255)
    return y, W


def build_wiener():
    rng = np.random.default_rng(20260101)
    cases = []
    specs = [("constant", np.full((6, 7), 91, np.uint8), 3),
             ("ramp5x5", (np.arange(25).reshape(5, 5) * 10).astype(np.uint8), 3),
             ("impulse", np.pad(np.full((1, 1), 255, np.uint8), 3, constant_values=40), 3),
             ("checker", (np.indices((8, 8)).sum(0) % 2 * 200 + 20).astype(np.uint8), 5),
             ("random7", rng.integers(0, 256, (9, 11), dtype=np.uint8), 7),
             ("random3", rng.integers(0, 256, (13, 6), dtype=np.uint8), 3),
             ("row", rng.integers(0, 256, (1, 17), dtype=np.uint8), 5),
             ("col", rng.integers(0, 256, (15, 1), dtype=np.uint8), 3)]
    for name, f, win in specs:
        y, W = wiener_exact(f, win)
        cases.append({"name": name, "win": win, "f": f.tolist(), "y": y.tolist(), "W": W})
    return cases


def build_window_stats():
    """window_stats planes from the reference (proj/src/adaptive_median.cpp:96-119): its unit-test images
    (proj/tests/test_adaptive_median.cpp:26-59, rank-compressed / quantised) and random S&P images."""
    cases = {}

    def add(name, img, ks):
        cases[f"{name}/input"] = img
        for k in ks:
            zmin, zmed, zmax = oracle.ref_window_stats(img, k)
            cases[f"{name}/k{k}"] = np.stack([zmin, zmed, zmax])

    add("kat_ramp3", np.arange(1, 10, dtype=np.uint8).reshape(3, 3), [3, 5])
    add("kat_flat6x5", np.full((6, 5), 64, np.uint8), [5])
    add("random_21x17_99", oracle.ref_random_image(21, 17, 99, 0.0, 100), [3, 5, 7])
    for i, (rows, cols) in enumerate([(1, 1), (1, 40), (40, 1), (33, 70), (64, 48)]):
        img = oracle.ref_random_image(rows, cols, 900 + i, 0.3, 950 + i)
        add(f"sp_{rows}x{cols}", img, [3, 7, 11])
    return cases


def phantom_pins():
    """Reference Rng64 streams used by the BASELINE phantom generator (checked in test_phantom.py)."""
    return {
        "uniform_seed7": oracle.ref_rng(7, 16).tolist(),
        "normal_seed7": oracle.ref_rng(7, 16, normal=True).tolist(),
        "u64_seed1000": [str(v) for v in oracle.ref_rng_u64(1000, 4)],
        "salt_pepper_100x100_d005_seed77": oracle.ref().ref_salt_pepper_count(100, 100, 0.5, 0.05, 77),
    }


def main():
    if not oracle.ref_available():
        sys.exit("oracle/_ref/libref.so missing: run `make -C oracle` where /root/reference exists")
    if sys.argv[1:] == ["window_stats"]:  # only the window_stats fixture
        np.savez_compressed(os.path.join(HERE, "window_stats_reference.npz"), **build_window_stats())
        print("wrote window_stats_reference.npz")
        return
    amf = build_amf()
    np.savez_compressed(os.path.join(HERE, "amf_reference.npz"), **amf)
    np.savez_compressed(os.path.join(HERE, "window_stats_reference.npz"), **build_window_stats())
    with open(os.path.join(HERE, "wiener_kat.json"), "w") as fh:
        json.dump(build_wiener(), fh)
    with open(os.path.join(HERE, "rng_pins.json"), "w") as fh:
        json.dump(phantom_pins(), fh, indent=1)
    print(f"wrote {len(amf)} AMF arrays, W1 KATs, RNG pins")


if __name__ == "__main__":
    main()
