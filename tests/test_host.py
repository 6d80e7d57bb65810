"""CPU: host-side logic of the strip partitioner and the reference-API mirror."""
import numpy as np
import pytest

import oracle
from paper_2005_05371_b200 import FilterConfig, denoise, split_bands, validate_config, validate_smax
from paper_2005_05371_b200.capi import InvalidArgument
from paper_2005_05371_b200.partition import StripPlan


def test_validate_smax_messages():
    validate_smax(3)
    validate_smax(11)
    for bad in (4, 1, 0, -3):
        with pytest.raises(InvalidArgument, match="odd integer > 1"):
            validate_smax(bad)


def test_validate_config():
    validate_config(FilterConfig(smax=11, parts=4, workers=4))
    with pytest.raises(InvalidArgument):
        validate_config(FilterConfig(smax=4))
    with pytest.raises(InvalidArgument, match="parts must be >= 1"):
        validate_config(FilterConfig(smax=3, parts=0))
    with pytest.raises(InvalidArgument, match="workers must be >= 1"):
        validate_config(FilterConfig(smax=3, workers=0))


def test_split_bands_enumerated():
    # proj/tests/test_image_core.cpp:149-173 (8 rows, 4 parts, halo 1)
    b = split_bands(8, 4, 1)
    assert [(t.core_start, t.core_rows) for t in b] == [(0, 2), (2, 2), (4, 2), (6, 2)]
    assert (b[0].halo_above, b[0].halo_below) == (0, 1)
    assert (b[1].halo_above, b[1].halo_below) == (1, 1)
    assert (b[3].halo_above, b[3].halo_below) == (1, 0)
    with pytest.raises(InvalidArgument):
        split_bands(5, 6, 0)
    with pytest.raises(InvalidArgument):
        split_bands(5, 2, -1)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_split_bands_matches_reference():
    for rows in (1, 2, 7, 8, 63, 100, 1600):
        for parts in range(1, min(rows, 13) + 1):
            for halo in (0, 1, 2, 5, 20):
                ours = [(t.core_start, t.core_rows, t.halo_above, t.halo_below) for t in split_bands(rows, parts, halo)]
                assert ours == oracle.ref_split_bands(rows, 4, parts, halo)


def test_strip_plan_covers_rows_once():
    for rows, world, smax, win in [(1600, 2, 7, 3), (1600, 8, 7, 3), (8192, 8, 9, 5), (16384, 8, 11, 7), (97, 4, 5, 5)]:
        plans = [StripPlan(rows, 64, smax, win, world, r) for r in range(world)]
        covered = np.zeros(rows, int)
        for p in plans:
            covered[p.core_slice()] += 1
            assert p.g_rows == p.hA + p.core + p.hB
            assert p.fa <= p.hA and p.fb <= p.hB
            assert p.hA == min(p.h, p.start)
        assert (covered == 1).all()


def test_uint8_reference_grid_roundtrip():
    u = np.arange(256, dtype=np.uint8).reshape(16, 16)
    np.testing.assert_array_equal(denoise.to_u8(denoise.to_unit(u)), u)
    with pytest.raises(InvalidArgument):
        denoise.to_u8(np.array([[0.1234]]))
