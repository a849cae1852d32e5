"""The CPU oracle (oracle/) against golden vectors from the unmodified reference.

Pins the oracle before anything is checked against it (task ③): every golden vector in
tests/golden/ was produced by wavehop 0.1.0 itself (oracle/gen_golden.py).  Tolerances
follow the reference's own tests: 1e-12 for direct/fold paths (test_kernels.py:21-61,
test_wavelet.py:169-174), 1e-9 for FFT-routed rows (test_wavelet.py:245-252).
"""
import math

import numpy as np
import pytest

from conftest import golden_cases, max_rel_err
from oracle import oracle as O


def test_half_widths_every_config(golden_taps):
    # wavelet.py:154 ceil in float64 -- bit-exact integer per scale
    for c in range(1, 6):
        got = np.array([O.half_width(s) for s in golden_taps[f"scales_c{c}"]])
        np.testing.assert_array_equal(got, golden_taps[f"half_c{c}"])


def test_taps_match_reference(golden_taps):
    for i, s in enumerate(golden_taps["pick_scales"]):
        ref = golden_taps[f"taps_{i}"]
        got = O.sample_wavelet(float(s))
        assert got.shape == ref.shape
        assert max_rel_err(got, ref) <= 1e-14


def test_taps_alt_params(golden_taps):
    C, B, R = golden_taps["alt_params"]
    for i, s in enumerate(golden_taps["alt_scales"]):
        ref = golden_taps[f"alt_taps_{i}"]
        got = O.sample_wavelet(float(s), C, B, R)
        assert got.shape == ref.shape
        assert max_rel_err(got, ref) <= 1e-14


def test_center_tap_closed_form():
    # test_wavelet.py:88-94
    for a in (1.0, 4.0, 37.5):
        t = O.sample_wavelet(a)
        c = t.size // 2
        assert t[c].real == pytest.approx((math.pi * 1.5) ** -0.5 / math.sqrt(a), rel=1e-15)
        assert t[c].imag == 0.0


def test_every_golden_transform(golden_cwth):
    for case in golden_cases(golden_cwth):
        got = O.cwth_batch(case["x"], case["scales"], case["hop"], output="complex",
                           center_frequency=case["C"], bandwidth=case["B"], support_radius=case["R"])
        assert got.shape == case["ref"].shape, case["name"]
        assert max_rel_err(got, case["ref"]) <= 1e-12, case["name"]


def test_frame_counts(golden_cwth):
    # wavelet.py:238: frames = ceil(N / hop) -- and the paper-scale case 160000/128 -> 1250
    for case in golden_cases(golden_cwth):
        assert case["ref"].shape[1] == -(-case["x"].size // case["hop"])
    assert -(-160_000 // 128) == 1250


def test_impulse_sifts_the_wavelet_exactly(golden_cwth):
    # test_wavelet.py:156-167: a unit impulse at n0 reproduces the taps exactly
    for name, hop in (("impulse_h1", 1), ("impulse_h4", 4)):
        x = golden_cwth[f"{name}__x"]
        sc = golden_cwth[f"{name}__scales"]
        n0 = int(np.argmax(x))
        out = O.cwth_batch(x, sc, hop, output="complex")
        for row, a in enumerate(sc):
            taps = O.sample_wavelet(a)
            c = taps.size // 2
            assert out[row, n0 // hop] == taps[c]
            for b in (n0 - 8, n0 + 4):
                if b % hop == 0:
                    assert out[row, b // hop] == taps[c + n0 - b]


def test_folded_kernel_matches_generic():
    # _kernels.py:93-112 vs 76-91 (test_kernels.py:47-61)
    rng = np.random.default_rng(3)
    for hop, half, frames in [(1, 4, 30), (9, 100, 21), (128, 513, 7)]:
        width = 2 * half + 1
        xpad = rng.standard_normal((frames - 1) * hop + width + 2)
        even = rng.standard_normal(half + 1)
        odd = np.concatenate([[0.0], rng.standard_normal(half)])
        taps_re = np.concatenate([even[:0:-1], even])
        taps_im = np.concatenate([-odd[:0:-1], odd])
        f = O.strided_correlate_symmetric(xpad, even, odd, hop, frames)
        g = O.strided_correlate(xpad, taps_re, taps_im, hop, frames)
        scale = max(np.abs(g[0]).max(), np.abs(g[1]).max())
        np.testing.assert_allclose(f[0], g[0], rtol=0, atol=1e-12 * scale)
        np.testing.assert_allclose(f[1], g[1], rtol=0, atol=1e-12 * scale)


def test_numpy_polyphase_port_matches_loop():
    # _kernels.py:28-62 vs a plain loop (test_kernels.py:21-30)
    rng = np.random.default_rng(5)
    for hop, width, frames in [(1, 7, 50), (3, 33, 40), (16, 129, 25)]:
        xpad = rng.standard_normal((frames - 1) * hop + width + 5)
        tr, ti = rng.standard_normal(width), rng.standard_normal(width)
        got = O.strided_correlate_numpy(xpad, tr, ti, hop, frames)
        want = O.strided_correlate(xpad, tr, ti, hop, frames)
        np.testing.assert_allclose(got[0], want[0], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(got[1], want[1], rtol=1e-12, atol=1e-12)


def test_routed_port_matches_reference(golden_cwth):
    # the FFT row route (wavelet.py:249,257-260,313-323) used for the CPU baseline
    for name in ("c3s", "c2s", "c5s"):
        x = golden_cwth[f"{name}__x"]
        sc = golden_cwth[f"{name}__scales"]
        hop = int(golden_cwth[f"{name}__meta"][0])
        got = O.cwth_strided_routed(x.astype(np.float64), sc, hop)
        assert max_rel_err(got, golden_cwth[f"{name}__ref"]) <= 1e-9
        got_np = O.cwth_strided_routed(x.astype(np.float64), sc, hop, backend="numpy")
        assert max_rel_err(got_np, golden_cwth[f"{name}__ref"]) <= 1e-9


def test_magnitude_modes_match_reference(golden_cwth):
    ref = golden_cwth["c5s__ref"]
    np.testing.assert_allclose(O.epilogue(ref, "cmor", "abs"), golden_cwth["mag_abs"], rtol=1e-15)
    np.testing.assert_allclose(O.epilogue(ref, "cmor", "power"), golden_cwth["mag_power"], rtol=1e-14)
    np.testing.assert_allclose(O.epilogue(ref, "cmor", "log_db"), golden_cwth["mag_log_db"], rtol=1e-14)
    # scalogram.py:64 pins zeros to exactly -240 dB; test_scalogram.py:41-51 (3+4j -> 5 / 25)
    assert O.epilogue(np.zeros((1, 1), complex), "cmor", "log_db")[0, 0] == -240.0
    z = np.array([[3 + 4j]])
    assert O.epilogue(z, "cmor", "abs")[0, 0] == 5.0 and O.epilogue(z, "cmor", "power")[0, 0] == 25.0


def test_batch_epilogues_match_per_clip(golden_cwth):
    x = golden_cwth["c5s__x"]
    sc = golden_cwth["c5s__scales"]
    ref = golden_cwth["c5s__ref"]
    for wavelet in ("cmor", "rmor"):
        for output in ("abs", "power", "log_db", "log1p"):
            for norm in (None, "minmax"):
                got = O.cwth_batch(x, sc, 32, wavelet=wavelet, output=output, norm=norm)
                want = O.epilogue(ref, wavelet, output, norm)
                np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-12)


def test_minmax_constant_clip_is_zero(golden_cwth):
    out = O.cwth_batch(golden_cwth["zeros__x"], golden_cwth["zeros__scales"], 16, output="abs",
                       norm="minmax")
    assert np.all(out == 0.0)


def test_oracle_threads_bit_identical(golden_cwth):
    # test_wavelet.py:274-279: row concurrency does not change results
    x = np.stack([golden_cwth["c2s__x"]] * 3)
    sc = golden_cwth["c2s__scales"]
    a = O.cwth_batch(x, sc, 64, output="complex", threads=1)
    b = O.cwth_batch(x, sc, 64, output="complex", threads=5)
    np.testing.assert_array_equal(a, b)


def test_oracle_errors():
    with pytest.raises(ValueError):
        O.cwth_batch(np.zeros(10, np.float32), [1.0], 0)
    with pytest.raises(ValueError):
        O.cwth_batch(np.zeros(10, np.float32), [0.0], 1)


def test_nonfinite_fixture_follows_the_support_rule():
    """tests/golden/nonfinite.npz (the reference's outputs on NaN / inf inputs): the non-finite
    coefficients are exactly those whose support holds a non-finite sample."""
    import math
    import os

    from conftest import GOLDEN

    g = np.load(os.path.join(GOLDEN, "nonfinite.npz"))
    names = sorted({k.split("__")[0] for k in g.files})
    assert len(names) == 6
    for n in names:
        x, sc, hop, ref = g[f"{n}__x"], g[f"{n}__scales"], int(g[f"{n}__hop"]), g[f"{n}__ref"]
        bad = np.where(~np.isfinite(x))[0]
        k = np.arange(ref.shape[1])
        for s, a in enumerate(sc):
            L = math.ceil(6.0 * a * math.sqrt(0.75))
            exp = np.zeros(ref.shape[1], bool)
            for t in bad:
                exp |= np.abs(k * hop - t) <= L
            np.testing.assert_array_equal(~np.isfinite(ref[s]), exp)
