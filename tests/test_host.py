"""Host-side logic that needs no GPU: parameter types, validation, synthetic inputs,
sharding arithmetic and bench bookkeeping."""
import math

import numpy as np
import pytest

import bench
from paper_2408_14302_b200 import (CoefficientMatrix, EmptySignal, InvalidCount, InvalidHop,
                                   InvalidRange, InvalidScale, MorletParams, ScaleGrid, SignalBuffer,
                                   make_scale_grid, scale_to_frequency, synth)
from paper_2408_14302_b200.shard import shard_range
from paper_2408_14302_b200.signal_io import _check_hop


def test_signal_buffer_validation():
    s = SignalBuffer([1, 2, 3], 16000)
    assert s.samples.dtype == np.float64 and len(s) == 3 and s.duration == 3 / 16000
    with pytest.raises(EmptySignal):
        SignalBuffer([], 16000)
    with pytest.raises(ValueError):
        SignalBuffer(np.zeros((2, 2)), 16000)
    with pytest.raises(ValueError):
        SignalBuffer([1.0], 0.0)


def test_check_hop_mirrors_reference():
    assert _check_hop(3) == 3 and _check_hop(4.0) == 4
    for bad in (0, -1, 1.5):
        with pytest.raises(InvalidHop):
            _check_hop(bad)
    assert issubclass(InvalidHop, ValueError)


def test_param_types():
    MorletParams()
    for kw in ({"center_frequency": 0}, {"bandwidth": -1}, {"support_radius": 2.9}):
        with pytest.raises(ValueError):
            MorletParams(**kw)
    with pytest.raises(ValueError):
        ScaleGrid([2.0, 1.0])
    with pytest.raises(ValueError):
        ScaleGrid([])
    with pytest.raises(ValueError):
        ScaleGrid([-1.0, 1.0])
    g = ScaleGrid([1.0, 2.0])
    assert g.count == 2
    with pytest.raises(InvalidHop):
        CoefficientMatrix(np.zeros((2, 4), complex), 0, 16000.0, g)
    with pytest.raises(ValueError):
        CoefficientMatrix(np.zeros((3, 4), complex), 1, 16000.0, g)


def test_scale_grid_and_frequency():
    # test_wavelet.py:59-84, 131-132
    np.testing.assert_array_equal(make_scale_grid(1000.0, 1000.0, 1, 16000.0).scales, [16.0])
    assert scale_to_frequency(16.0, MorletParams(), 16000.0) == 1000.0
    with pytest.raises(InvalidRange):
        make_scale_grid(100.0, 8000.0, 8, 16000.0)
    with pytest.raises(InvalidCount):
        make_scale_grid(100.0, 200.0, 1, 16000.0)
    with pytest.raises(InvalidScale):
        scale_to_frequency(-1.0, MorletParams(), 16000.0)


def test_synth_deterministic_and_shaped():
    a = synth.make_clip(2, 5, 4000)
    b = synth.make_clip(2, 5, 4000)
    c = synth.make_clip(2, 6, 4000)
    assert a.dtype == np.float32 and a.shape == (4000,)
    np.testing.assert_array_equal(a, b)
    assert not np.array_equal(a, c)
    c1 = synth.make_clip(1, 0)
    assert c1.shape == (16000,)
    batch = synth.make_batch(5, clips=3, n=1000, start=7)
    np.testing.assert_array_equal(batch[1], synth.make_clip(5, 8, 1000))


def test_config_scales_match_baseline():
    for cid, (a0, a1, s) in [(1, (1, 64, 32)), (2, (1, 128, 128)), (3, (1, 128, 64)),
                             (4, (1, 256, 64)), (5, (1, 512, 160))]:
        sc = synth.config_scales(cid)
        assert sc.size == s and sc[0] == a0 and math.isclose(sc[-1], a1)
        assert np.all(np.diff(sc) > 0)


def test_shard_range_partitions():
    for n in (0, 1, 7, 64, 4096):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(n, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def test_bench_workloads_and_flops():
    w = bench.workload("c2")
    assert w["clips"] == 64 and w["hop"] == 64 and w["wavelet"] == "rmor" and w["output"] == "log1p"
    assert bench.coeffs(w, 64) == 64 * 128 * 2500
    # W_alg = clips * F * 2 * sum(2L+1): c2 sum T = 35,468
    assert bench.alg_flops(w, 1) == 2500 * 2 * 35468
    w5 = bench.workload("c5")
    assert w5["scaling"] == "strong" and w5["wavelet"] == "cmor" and w5["norm"] == "minmax"
    assert bench.alg_flops(w5, 1) == 5000 * 4 * 138342
    assert bench.workload("c4h1024")["hop"] == 1024
