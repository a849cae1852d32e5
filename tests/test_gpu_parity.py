"""GPU parity: the CUDA engines (through the C ABI) against the pinned CPU oracle and the
reference's golden vectors.  Run on a B200 with ``pytest -m gpu``.

Tolerances (written here once):
  * complex / |W| / power: per (clip, scale) row, max_k |out - ref| / max_k |ref_row|
    <= ROW_TOL = 1e-5 (power: 2e-5, it squares the relative error);
  * log1p: absolute <= 1e-5; log_db: absolute <= 20/ln10 * 1e-5 + 2e-5 (dB);
  * per-clip min-max: absolute <= 1e-5 * max/(max - min) (+ the fast-log term);
  * bit-exact: shapes (B, S, ceil(N/hop)), frame k <-> sample k*hop, scale order,
    the impulse KAT on the SIMT engine, sharded == unsharded bytes.
"""
import ctypes
import math

import numpy as np
import pytest
import torch

import paper_2408_14302_b200 as wh
from conftest import golden_cases, row_rel_err
from oracle import oracle as O
from paper_2408_14302_b200 import _lib, synth
from paper_2408_14302_b200.shard import cwth_multi_device, shard_range

pytestmark = pytest.mark.gpu

ROW_TOL = 1e-5
ENGINES = ("umma", "simt")


def umma_ok(hop):
    # rows of lcm(hop, 64) <= 192 samples (hop | 64, hop | 192, 128), or, from 256, rows of 128
    # samples of which every (hop/128)-th is a frame (multiples of 128)
    return (math.lcm(hop, 64) <= 256 and hop < 256) or (hop >= 256 and hop % 128 == 0)


def engines_for(hop):
    return [e for e in ENGINES if e == "simt" or umma_ok(hop)]


def gpu(x, scales, hop, engine, params=None, **kw):
    return wh.cwth_batch(np.asarray(x, np.float32), scales, params or wh.MorletParams(), hop,
                         engine=engine, **kw)


# ---------------------------------------------------------------------------------------
# golden vectors (the reference's own outputs)
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("engine", ENGINES)
def test_golden_cases_complex(golden_cwth, engine):
    for case in golden_cases(golden_cwth):
        if not (engine == "simt" or umma_ok(case["hop"])):
            continue
        p = wh.MorletParams(case["C"], case["B"], case["R"])
        got = gpu(case["x"][None], case["scales"], case["hop"], engine, p, output="complex")[0]
        ref = case["ref"]
        assert got.shape == ref.shape, case["name"]
        assert row_rel_err(got, ref) <= ROW_TOL, (case["name"], row_rel_err(got, ref))


@pytest.mark.parametrize("engine", ENGINES)
def test_golden_real_morlet_configs(golden_cwth, engine):
    """c1 (full BASELINE config 1) and the small c2-c4 cases as real Morlet |W|."""
    for name in ("c1", "c2s", "c3s", "c4s_h16", "c4s_h256", "c4s_h1024"):
        hop = int(golden_cwth[f"{name}__meta"][0])
        if engine == "umma" and not umma_ok(hop):
            continue
        ref = np.abs(golden_cwth[f"{name}__ref"].real)
        got = gpu(golden_cwth[f"{name}__x"][None], golden_cwth[f"{name}__scales"], hop, engine,
                  wavelet="rmor", output="abs")[0]
        assert row_rel_err(got, ref) <= ROW_TOL, name


def test_device_taps_within_one_ulp(golden_taps):
    """The on-device filter-bank builder (fp64 math, fp32 store) vs sample_wavelet."""
    for i, s in enumerate(golden_taps["pick_scales"]):
        ref = golden_taps[f"taps_{i}"]
        got = wh.sample_wavelet(wh.MorletParams(), float(s))
        assert got.shape == ref.shape  # 2L+1 taps: L bit-exact
        r32 = ref.astype(np.complex64)
        ulp = np.spacing(np.abs(r32.real).astype(np.float32).max())
        assert np.abs(got.real - r32.real).max() <= np.spacing(np.abs(r32.real)).max() + ulp
        assert np.abs(got.imag - r32.imag).max() <= np.spacing(np.abs(r32.imag)).max() + ulp


@pytest.mark.parametrize("engine", ENGINES)
def test_impulse_sifts_the_wavelet(golden_cwth, engine):
    """test_wavelet.py:156-167: out[row, n0/hop] == taps[center] (exact on SIMT: 1.0 x tap)."""
    for name, hop in (("impulse_h1", 1), ("impulse_h4", 4)):
        x = golden_cwth[f"{name}__x"]
        sc = golden_cwth[f"{name}__scales"]
        n0 = int(np.argmax(x))
        out = gpu(x[None], sc, hop, engine, output="complex")[0]
        for row, a in enumerate(sc):
            taps = wh.sample_wavelet(wh.MorletParams(), float(a)).astype(np.complex64)
            c = taps.size // 2
            if engine == "simt":
                assert out[row, n0 // hop] == taps[c]
            else:
                assert abs(out[row, n0 // hop] - taps[c]) <= 1e-6 * abs(taps[c])


# ---------------------------------------------------------------------------------------
# fused epilogues vs the oracle
# ---------------------------------------------------------------------------------------

def minmax_tol(raw, output):
    """Per clip: the normalised map's absolute tolerance from the un-normalised values' own
    (SURVEY.md App. B): 1e-5 * max/(max - min) for |W| (a relative error of the magnitudes),
    2e-5 * max/(max - min) for power, 1e-5/(max - min) for log1p (an absolute error)."""
    raw = np.asarray(raw, np.float64).reshape(raw.shape[0], -1)
    hi, lo = raw.max(axis=1), raw.min(axis=1)
    span = np.where(hi > lo, hi - lo, np.inf)
    if output == "log1p":
        return 1e-5 / span
    if output == "log_db":
        return (20.0 / np.log(10.0) * 1e-5 + 2e-5) / span
    return (2e-5 if output == "power" else 1e-5) * np.abs(hi) / span


def check_minmax(got, ref, raw, output):
    assert np.all(got >= -1e-6) and np.all(got <= 1 + 1e-6)
    err = np.abs(got.astype(np.float64) - ref).reshape(got.shape[0], -1).max(axis=1)
    tol = minmax_tol(raw, output)
    assert np.all(err <= tol), (err, tol)


def check_output(got, ref, output, norm, raw=None):
    if norm == "minmax":
        check_minmax(got, ref, raw, output)
    elif output == "log1p":
        assert np.abs(got - ref).max() <= 1e-5
    elif output == "log_db":
        # dB amplifies relative error near |W| = 0; compare the magnitudes it encodes
        to_mag = lambda d: 10.0 ** (np.asarray(d, np.float64) / 20.0)  # noqa: E731
        assert row_rel_err(to_mag(got), to_mag(ref)) <= ROW_TOL + 2e-6
    elif output == "power":
        assert row_rel_err(got, ref) <= 2 * ROW_TOL
    else:
        assert row_rel_err(got, ref) <= ROW_TOL


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("wavelet", ["cmor", "rmor"])
@pytest.mark.parametrize("output,norm", [("abs", None), ("power", None), ("log1p", None),
                                         ("log_db", None), ("abs", "minmax"), ("log1p", "minmax")])
def test_epilogues_match_oracle(engine, wavelet, output, norm):
    x = synth.make_batch(5, clips=3, n=6000, start=11)
    sc = np.geomspace(1, 512, 12)
    got = gpu(x, sc, 32, engine, wavelet=wavelet, output=output, norm=norm)
    ref = O.cwth_batch(x, sc, 32, wavelet=wavelet, output=output, norm=norm)
    raw = O.cwth_batch(x, sc, 32, wavelet=wavelet, output=output) if norm else None
    assert got.shape == ref.shape
    check_output(got, ref, output, norm, raw)


# ---------------------------------------------------------------------------------------
# BASELINE configurations at full size
# ---------------------------------------------------------------------------------------

def cfg_run(cid, clips, hop=None, engine="auto", start=0):
    cfg = synth.CONFIGS[cid]
    hop = hop or cfg["hop"]
    x = synth.make_batch(cid, clips=clips, start=start)
    sc = synth.config_scales(cid)
    got = gpu(x, sc, hop, engine, wavelet=cfg["wavelet"], output=cfg["output"], norm=cfg["norm"])
    return x, sc, hop, cfg, got


def test_c2_full_batch_parity():
    """BASELINE config 2 at full size: 64 clips x 160,000 samples, 128 scales, hop 64, log1p."""
    x, sc, hop, cfg, got = cfg_run(2, 64)
    assert got.shape == (64, 128, 2500)
    ref = O.cwth_batch(x, sc, hop, wavelet="rmor", output="log1p")
    assert np.abs(got - ref).max() <= 1e-5


def test_c3_full_hop1_parity():
    """BASELINE config 3 (full CWT, hop 1): all 8 clips x 160,000 x 64 scales vs the oracle."""
    x, sc, hop, cfg, got = cfg_run(3, 8)
    assert got.shape == (8, 64, 160000)
    ref = O.cwth_batch(x, sc, 1, wavelet="rmor", output="abs")
    assert row_rel_err(got, ref) <= ROW_TOL


@pytest.mark.parametrize("hop", [1, 16, 64, 256, 1024])
def test_c4_hop_sweep_parity(hop):
    """BASELINE config 4 sweep: 2 clips per hop vs the oracle; frames = ceil(N/hop)."""
    x, sc, hop, cfg, got = cfg_run(4, 2, hop=hop)
    assert got.shape == (2, 64, -(-160000 // hop))
    ref = O.cwth_batch(x, sc, hop, wavelet="rmor", output="abs")
    assert row_rel_err(got, ref) <= ROW_TOL


@pytest.mark.parametrize("hop", [16, 64, 256, 1024])
def test_c4_full_launch_sampled_clips(hop):
    """The 256-clip c4 launch the sweep times (unit counts, clip offsets and 32-bit index math at
    full size): clips 0, 131 and 255 of the one launch against the oracle."""
    from concurrent.futures import ThreadPoolExecutor

    x = np.empty((256, 160000), np.float32)
    with ThreadPoolExecutor(16) as ex:
        list(ex.map(lambda c: x.__setitem__(c, synth.make_clip(4, c)), range(256)))
    sc = synth.config_scales(4)
    plan = wh.CwthPlan(sc, None, hop, 160000, wavelet="rmor", output="abs", max_clips=256, engine="umma")
    out = plan.execute(torch.from_numpy(x).cuda())
    ids = [0, 131, 255]
    got = out[ids].cpu().numpy()
    plan.close()
    ref = O.cwth_batch(x[ids], sc, hop, wavelet="rmor", output="abs", threads=16)
    assert row_rel_err(got, ref) <= ROW_TOL


def test_c4_hop_columns_are_full_transform_columns():
    """test_wavelet.py:245-252 at BASELINE size: cwth(hop)[:, k] == cwth(1)[:, k*hop]."""
    x = synth.make_batch(4, clips=1, start=3)
    sc = synth.config_scales(4)
    full = gpu(x, sc, 1, "auto", wavelet="rmor", output="complex")[0]
    for hop in (16, 64, 256, 1024):
        hopped = gpu(x, sc, hop, "auto", wavelet="rmor", output="complex")[0]
        assert hopped.shape[1] == -(-160000 // hop)
        assert row_rel_err(hopped, full[:, ::hop]) <= 2 * ROW_TOL


def test_c5_sample_parity_and_minmax_range():
    """BASELINE config 5 (complex Morlet, 160 scales 1-512, hop 32, per-clip min-max)."""
    x, sc, hop, cfg, got = cfg_run(5, 4)
    assert got.shape == (4, 160, 5000)
    ref = O.cwth_batch(x, sc, hop, wavelet="cmor", output="abs", norm="minmax")
    raw = O.cwth_batch(x, sc, hop, wavelet="cmor", output="abs")
    check_minmax(got, ref, raw, "abs")
    for c in range(4):
        assert got[c].min() == 0.0 and abs(got[c].max() - 1.0) <= 1e-6


def test_c5_full_launch_4096_clips():
    """The launch the bench times: all 4096 c5 clips in one wh_execute.  Every clip's
    normalised scalogram spans exactly [0, 1] (per-clip min-max), and clips 0,
    2048 and 4095 match the oracle (32-bit unit math, clip counters and min-max slices at full
    size)."""
    cfg = synth.CONFIGS[5]
    from concurrent.futures import ThreadPoolExecutor

    x = np.empty((4096, 160000), np.float32)
    with ThreadPoolExecutor(16) as ex:
        list(ex.map(lambda c: x.__setitem__(c, synth.make_clip(5, c)), range(4096)))
    sc = synth.config_scales(5)
    plan = wh.CwthPlan(sc, None, 32, 160000, wavelet="cmor", output="abs", norm="minmax",
                       max_clips=4096, engine="umma")
    xd = torch.from_numpy(x).cuda()
    out = plan.execute(xd)
    torch.cuda.synchronize()
    flat = out.view(4096, -1)
    assert torch.all(flat.amin(dim=1) == 0.0)
    assert torch.all((flat.amax(dim=1) - 1.0).abs() <= 1e-6)
    ids = [0, 2048, 4095]
    got = out[ids].cpu().numpy()
    plan.close()
    ref = O.cwth_batch(x[ids], sc, 32, wavelet="cmor", output="abs", norm="minmax", threads=16)
    raw = O.cwth_batch(x[ids], sc, 32, wavelet="cmor", output="abs", threads=16)
    check_minmax(got, ref, raw, "abs")


@pytest.mark.parametrize("output", ["abs", "log1p"])
def test_write_once_minmax_fixup_path_is_byte_identical(output, monkeypatch):
    """The write-once variant (WH_UMMA_MINMAX_INKERNEL=1): units the kernel could not normalise itself (their clip still running elsewhere
    after a bounded wait) go to the fix-up kernel; forcing every unit down that path
    (WH_UMMA_MINMAX_FIXUP=1, a planner override) gives byte-identical output, and both match
    the SIMT engine's read-modify-write pass within tolerance."""
    monkeypatch.setenv("WH_UMMA_MINMAX_INKERNEL", "1")  # the write-once variant (planner option)
    x = synth.make_batch(5, clips=5, n=50000, start=7)
    sc = synth.config_scales(5)
    mk = lambda: wh.CwthPlan(sc, None, 32, 50000, wavelet="cmor", output=output, norm="minmax",  # noqa: E731
                             max_clips=5, engine="umma")
    plan = mk()
    inkernel = plan.execute_host(x).copy()
    plan.close()
    monkeypatch.setenv("WH_UMMA_MINMAX_FIXUP", "1")
    plan = mk()
    fixup = plan.execute_host(x).copy()
    assert plan.launches(5) == 3
    plan.close()
    assert inkernel.tobytes() == fixup.tobytes()
    monkeypatch.delenv("WH_UMMA_MINMAX_INKERNEL")
    monkeypatch.delenv("WH_UMMA_MINMAX_FIXUP")
    plan = mk()
    twopass = plan.execute_host(x).copy()  # the default: a separate read-modify-write pass
    plan.close()
    assert twopass.tobytes() == inkernel.tobytes()
    ref = O.cwth_batch(x, sc, 32, wavelet="cmor", output=output, norm="minmax")
    raw = O.cwth_batch(x, sc, 32, wavelet="cmor", output=output)
    check_minmax(inkernel, ref, raw, output)


def test_near_silent_and_subnormal_amplitude_clips():
    """Window exponents are clamped so that 2^e and 2^-e stay finite normal floats: clips at
    1e-30 and 1e-38 of full scale (the latter near the fp32 subnormal range) still match the
    oracle's relative accuracy, and a clip with a single subnormal sample is finite."""
    base = synth.make_batch(2, clips=1, n=20000, start=5)[0].astype(np.float64)
    sc = synth.config_scales(2)
    for amp in (1e-30, 1e-38):
        x = (base * amp).astype(np.float32)[None]
        got = gpu(x, sc, 64, "umma", wavelet="rmor", output="abs")
        ref = O.cwth_batch(x, sc, 64, wavelet="rmor", output="abs")
        assert np.all(np.isfinite(got))
        assert row_rel_err(got, ref) <= ROW_TOL, amp
    x = np.zeros((1, 20000), np.float32)
    x[0, 777] = np.float32(1e-42)  # subnormal
    got = gpu(x, sc, 64, "umma", wavelet="rmor", output="abs")
    assert np.all(np.isfinite(got)) and got.max() > 0


# ---------------------------------------------------------------------------------------
# size-independent properties at full size
# ---------------------------------------------------------------------------------------

def test_linearity_full_size():
    """test_wavelet.py:326-346: W(a x + b y) = a W(x) + b W(y)."""
    x = synth.make_batch(5, clips=2, start=40)
    sc = synth.config_scales(5)
    a, b = 0.3, -0.7
    lhs = gpu((a * x[0] + b * x[1])[None], sc, 32, "auto", output="complex")[0]
    w = gpu(x, sc, 32, "auto", output="complex")
    assert row_rel_err(lhs, a * w[0] + b * w[1]) <= 3 * ROW_TOL


def test_sharded_equals_unsharded_bytes():
    """Per-clip work is identical, so any clip split gives byte-equal scalograms."""
    x = synth.make_batch(2, clips=10, start=0)
    sc = synth.config_scales(2)
    whole = gpu(x, sc, 64, "auto", wavelet="rmor", output="log1p")
    parts = [gpu(x[a:b], sc, 64, "auto", wavelet="rmor", output="log1p")
             for a, b in (shard_range(10, 3, r) for r in range(3))]
    np.testing.assert_array_equal(whole, np.concatenate(parts))
    multi = cwth_multi_device(x, sc, None, 64, devices=[0, 0], wavelet="rmor", output="log1p")
    np.testing.assert_array_equal(whole, multi)


def test_zero_signal_and_constant_minmax():
    sc = synth.config_scales(5)
    z = np.zeros((2, 160000), np.float32)
    assert np.all(gpu(z, sc, 32, "auto", output="abs") == 0.0)
    assert np.all(gpu(z, sc, 32, "auto", output="abs", norm="minmax") == 0.0)


def test_diagnostics_absent_from_product_build():
    """profile()/trace() need the WH_DIAG build; in the product library they fail loudly and
    leave the plan usable (the profile(False) path used to free the trace buffer the next
    launch wrote to)."""
    x = synth.make_batch(2, clips=1, n=8000)
    plan = wh.CwthPlan(np.geomspace(1, 32, 8), None, 16, 8000, wavelet="rmor", output="abs")
    before = plan.execute_host(x).copy()
    for call in (lambda: plan.profile(False), lambda: plan.trace(False)):
        with pytest.raises(wh.DeviceError):
            call()
    np.testing.assert_array_equal(plan.execute_host(x), before)
    plan.close()


def test_device_and_host_paths_identical():
    x = synth.make_batch(2, clips=3, n=20000)
    sc = np.geomspace(1, 128, 40)
    plan = wh.CwthPlan(sc, None, 64, 20000, wavelet="rmor", output="abs", max_clips=3)
    host = plan.execute_host(x)
    dev = plan.execute(torch.from_numpy(x).cuda()).cpu().numpy()
    np.testing.assert_array_equal(host, dev)
    assert plan.launches(3) == 1


@pytest.mark.parametrize("norm", [None, "minmax"])
def test_pageable_staged_and_pinned_host_paths_identical(norm):
    """wh_execute_host with pageable numpy buffers runs through the plan's pinned staging
    ring in clip chunks of ~64 MB (c2 shape: 33 clips per chunk, 100 clips = 4 chunks, the two
    slots recycled by events); the result is byte-identical to the pinned pipeline and to the
    device path."""
    n = 160000
    x = synth.make_batch(2, clips=100, n=n, start=3)
    sc = synth.config_scales(2)
    plan = wh.CwthPlan(sc, None, 64, n, wavelet="rmor", output="log1p", norm=norm, max_clips=100)
    pageable = plan.execute_host(x).copy()
    xpin = torch.from_numpy(x).pin_memory()
    opin = torch.empty(pageable.shape, dtype=torch.float32).pin_memory()
    plan.execute_host(xpin.numpy(), opin.numpy())
    dev = plan.execute(torch.from_numpy(x).cuda()).cpu().numpy()
    plan.close()
    assert pageable.tobytes() == opin.numpy().tobytes() == dev.tobytes()


# ---------------------------------------------------------------------------------------
# edges and errors
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("engine", ENGINES)
def test_ragged_and_tiny_signals(engine):
    rng = np.random.default_rng(9)
    for n, hop, scales in [(1001, 64, [1.0, 3.3, 20.0]), (5, 2, [1.0, 100.0]), (1, 1, [1.0, 2.0]),
                           (100, 128, [1.5, 6.0]), (4097, 16, [2.0, 64.0, 300.0])]:
        if engine == "umma" and not umma_ok(hop):
            continue
        x = rng.standard_normal((2, n)).astype(np.float32)
        got = gpu(x, scales, hop, engine, output="complex")
        ref = O.cwth_batch(x, scales, hop, output="complex")
        assert got.shape == ref.shape == (2, len(scales), -(-n // hop))
        assert row_rel_err(got, ref) <= ROW_TOL, (n, hop)


def test_engine_selection_and_errors():
    assert wh.CwthPlan([1.0, 2.0], None, 64, 1000).engine == "umma"
    assert wh.CwthPlan([1.0, 2.0], None, 1024, 5000).engine == "umma"  # rows of 256, every 4th a frame
    assert wh.CwthPlan([1.0, 2.0], None, 7, 1000).engine == "simt"
    assert wh.CwthPlan([1.0, 2.0], None, 320, 5000).engine == "umma"  # panel streaming (rows of 320)
    assert wh.CwthPlan([1.0, 2.0], None, 100, 5000).engine == "simt"
    with pytest.raises(wh.DeviceError):
        wh.CwthPlan([1.0, 2.0], None, 7, 1000, engine="umma")
    with pytest.raises(wh.InvalidHop):
        wh.CwthPlan([1.0], None, 0, 100)
    with pytest.raises(wh.InvalidScale):
        wh.CwthPlan([0.0, 1.0], None, 4, 100)
    with pytest.raises(ValueError):
        wh.CwthPlan([2.0, 1.0], None, 4, 100)
    plan = wh.CwthPlan([1.0, 2.0], None, 4, 100, max_clips=2)
    with pytest.raises(ValueError):
        plan.execute_host(np.zeros((3, 100), np.float32))
    with pytest.raises(ValueError):
        plan.execute_host(np.zeros((1, 99), np.float32))


def test_drop_in_signatures(golden_cwth):
    """cwth_strided / cwt_fft keep the reference signatures and metadata."""
    x = golden_cwth["c2s__x"]
    sc = golden_cwth["c2s__scales"]
    sig = wh.SignalBuffer(x.astype(np.float64), 16000.0)
    m = wh.cwth_strided(sig, wh.ScaleGrid(sc), wh.MorletParams(), 64, threads=4)
    assert m.hop == 64 and m.source_rate == 16000.0 and m.values.dtype == np.complex128
    assert m.columns == -(-x.size // 64) and m.rows == sc.size
    assert row_rel_err(m.values, golden_cwth["c2s__ref"]) <= ROW_TOL
    full = wh.cwt_fft(sig, wh.ScaleGrid(sc))
    assert full.hop == 1 and full.columns == x.size
    assert row_rel_err(full.values[:, ::64], m.values) <= 2 * ROW_TOL
    mag = wh.magnitude(m, "abs")
    assert row_rel_err(mag, np.abs(golden_cwth["c2s__ref"])) <= ROW_TOL


def test_seam2_kernels_match_oracle():
    """_kernels.py seam: float64 device kernels within 1e-12 of the oracle."""
    lib = _lib.load()
    rng = np.random.default_rng(2)
    for hop, half, frames in [(1, 4, 30), (9, 100, 21), (128, 513, 7)]:
        width = 2 * half + 1
        xpad = rng.standard_normal((frames - 1) * hop + width + 2)
        tr, ti = rng.standard_normal(width), rng.standard_normal(width)
        ore, oim = np.empty(frames), np.empty(frames)
        P = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        assert lib.wh_strided_correlate(0, P(xpad), xpad.size, P(tr), P(ti), width, hop, frames,
                                        P(ore), P(oim)) == 0
        r = O.strided_correlate(xpad, tr, ti, hop, frames)
        sc = max(np.abs(r[0]).max(), np.abs(r[1]).max())
        assert np.abs(ore - r[0]).max() <= 1e-12 * sc and np.abs(oim - r[1]).max() <= 1e-12 * sc
        even = rng.standard_normal(half + 1)
        odd = np.concatenate([[0.0], rng.standard_normal(half)])
        assert lib.wh_strided_correlate_symmetric(0, P(xpad), xpad.size, P(even), P(odd), half, hop,
                                                  frames, P(ore), P(oim)) == 0
        r = O.strided_correlate_symmetric(xpad, even, odd, hop, frames)
        sc = max(np.abs(r[0]).max(), np.abs(r[1]).max())
        assert np.abs(ore - r[0]).max() <= 1e-12 * sc and np.abs(oim - r[1]).max() <= 1e-12 * sc


@pytest.mark.parametrize("env", [{"WH_UMMA_HYBRID": "1"}, {"WH_UMMA_NO_RESIDENT": "1"},
                                 {"WH_UMMA_CG1": "1"}, {"WH_UMMA_TAU": "0"},
                                 {"WH_UMMA_NO_CONVREGS": "1"}, {"WH_UMMA_G0_ALIGN": "64"}])
def test_umma_planner_variants_agree(env, monkeypatch):
    """Every planner / kernel variant the diagnostics switches select (resident + streamed
    hybrid bank, fully streamed bank, single-CTA MMAs, no tail skipping, staged converter,
    another K origin) computes the same transform within tolerance (c2 and c5 shapes)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for cid, hop, wavelet, output in ((2, 64, "rmor", "log1p"), (5, 32, "cmor", "abs")):
        x = synth.make_batch(cid, clips=2, n=30000, start=4)
        sc = synth.config_scales(cid)
        plan = wh.CwthPlan(sc, None, hop, 30000, wavelet=wavelet, output=output, max_clips=2,
                           engine="umma")
        got = plan.execute_host(x)
        plan.close()
        ref = O.cwth_batch(x, sc, hop, wavelet=wavelet, output=output)
        if output == "log1p":
            assert np.abs(got - ref).max() <= 1e-5, env
        else:
            assert row_rel_err(got, ref) <= ROW_TOL, env


@pytest.mark.parametrize("hop,force", [(256, True), (1024, True), (320, False), (448, False)])
def test_panel_streaming_frames_only(hop, force, monkeypatch):
    """Rows of hop samples (one frame per row, the window streamed by 64-sample column panels
    through cp.async-filled slots, exponents from the segment-max pre-pass): the default for
    hops >= 256 that are multiples of 64 but not of 128, on request (WH_UMMA_PSTREAM=1) for
    the others -- against the oracle on c4-shaped clips, a NaN/inf clip included."""
    if force:
        monkeypatch.setenv("WH_UMMA_PSTREAM", "1")
    x = synth.make_batch(4, clips=3, n=60000, start=2)
    x[1, 12345] = np.inf
    x[1, 40000] = np.nan
    sc = synth.config_scales(4)
    plan = wh.CwthPlan(sc, None, hop, 60000, wavelet="rmor", output="abs", max_clips=3, engine="umma")
    got = plan.execute_host(x)
    plan.close()
    ref = O.cwth_batch(x[[0, 2]], sc, hop, wavelet="rmor", output="abs")
    assert row_rel_err(got[[0, 2]], ref) <= ROW_TOL
    # the bad clip: non-finite exactly on the supports (k*hop within L_s of 12345 / 40000)
    k = np.arange(got.shape[2])
    for s, a in enumerate(sc):
        L = math.ceil(6.0 * a * math.sqrt(0.75))
        want = (np.abs(k * hop - 12345) <= L) | (np.abs(k * hop - 40000) <= L)
        np.testing.assert_array_equal(~np.isfinite(got[1, s]), want)


@pytest.mark.parametrize("hop,tma", [(256, True), (1024, True), (2048, True), (320, False), (1024, False)])
def test_panel_streaming_tf32(hop, tma, monkeypatch):
    """Panel streaming with tf32 operands (WH_UMMA_TF32=1: kind::tf32 MMAs on 32-sample panels
    fetched by TMA tensor copies -- or cp.async with WH_UMMA_NO_TMA -- split in place into
    hi = the top 19 bits and lo = x - hi, two accumulator sets per buffer, no window exponent
    and no pre-pass): against the oracle on c4-shaped clips whose length is not a multiple of
    the hop (the clip's last partial row is patched from global memory), a NaN/inf clip and a
    tiny-amplitude clip (no exponent scaling: tf32 keeps fp32's range) included."""
    monkeypatch.setenv("WH_UMMA_PSTREAM", "1")
    monkeypatch.setenv("WH_UMMA_TF32", "1")
    if not tma:
        monkeypatch.setenv("WH_UMMA_NO_TMA", "1")
    n = 60000
    x = synth.make_batch(4, clips=4, n=n, start=2)
    x[1, 12345] = np.inf
    x[1, 40000] = np.nan
    x[3] *= np.float32(1e-30)
    sc = synth.config_scales(4)
    plan = wh.CwthPlan(sc, None, hop, n, wavelet="rmor", output="abs", max_clips=4, engine="umma")
    got = plan.execute_host(x)
    # rows that are not 16-byte aligned take the cp.async / scalar fetch whatever the knob says
    base = np.zeros((2, n + 7), np.float32)
    base[:, 3:3 + n] = x[[0, 2]]
    got_u = plan.execute(torch.from_numpy(base).cuda()[:, 3:3 + n]).cpu().numpy()
    plan.close()
    ref = O.cwth_batch(x[[0, 2, 3]], sc, hop, wavelet="rmor", output="abs")
    assert got.shape == (4, len(sc), -(-n // hop))
    assert row_rel_err(got[[0, 2, 3]], ref) <= ROW_TOL
    assert row_rel_err(got_u, ref[:2]) <= ROW_TOL
    k = np.arange(got.shape[2])
    for s, a in enumerate(sc):
        L = math.ceil(6.0 * a * math.sqrt(0.75))
        want = (np.abs(k * hop - 12345) <= L) | (np.abs(k * hop - 40000) <= L)
        np.testing.assert_array_equal(~np.isfinite(got[1, s]), want)


@pytest.mark.parametrize("engine,hop", [("umma", 32), ("umma", 1), ("umma", 4), ("simt", 20)])
def test_complex_magnitude_at_extreme_amplitudes(engine, hop):
    """|W| of the complex wavelet for clips scaled by 1e-25 and 1e+25: re^2 + im^2 would
    underflow to 0 / overflow to inf in float32 (the reference computes in float64); the
    epilogues take the root in a scaled domain, so the rows keep their relative accuracy."""
    n = 6000 if hop == 1 else 30000
    x = synth.make_batch(5, clips=3, n=n, start=5)
    x[1] *= np.float32(1e-25)
    x[2] *= np.float32(1e25)
    sc = synth.config_scales(5)[::4] if hop != 32 else synth.config_scales(5)
    plan = wh.CwthPlan(sc, None, hop, n, wavelet="cmor", output="abs", max_clips=3, engine=engine)
    got = plan.execute_host(x)
    plan.close()
    ref = O.cwth_batch(x, sc, hop, wavelet="cmor", output="abs")
    assert np.isfinite(got).all() and (got[1].max() > 0)
    assert row_rel_err(got, ref) <= ROW_TOL


@pytest.mark.parametrize("mode", ["inkernel", "concurrent"])
def test_minmax_modes_fall_back_where_their_kernel_variant_is_absent(mode, monkeypatch):
    """The opt-in min-max modes live in kernel variants of their own (CTA pairs, 1 or 2 phases
    per row, no panel streaming); plans of other shapes (hop 16: 4 phases; panel-streamed hop
    320) take the separate pass and give its bytes."""
    for hop, n in ((16, 20000), (320, 60000)):
        x = synth.make_batch(4, clips=3, n=n, start=7)
        sc = synth.config_scales(4)
        mk = lambda: wh.CwthPlan(sc, None, hop, n, wavelet="rmor", output="abs", norm="minmax",  # noqa: E731
                                 max_clips=3, engine="umma")
        monkeypatch.delenv("WH_UMMA_MINMAX", raising=False)
        plan = mk()
        want = plan.execute_host(x).copy()
        plan.close()
        monkeypatch.setenv("WH_UMMA_MINMAX", mode)
        plan = mk()
        got = plan.execute_host(x)
        plan.close()
        assert got.tobytes() == want.tobytes(), (mode, hop)


def test_very_long_taps():
    """The split-fp16 accumulation's row error grows with the taps per accumulator (the tensor
    core's fp32 accumulate truncates).  Half widths beyond 3,360 taps (scales above ~650) run
    with two accumulator sets per buffer (kernel variant 3, hops 16 / 32 / 64); beyond 5,632
    (scale ~1,080) -- or at other hops -- AUTO takes the SIMT engine and a forced UMMA plan is
    refused.  Every case within the row tolerance."""
    n = 48000
    x = synth.make_batch(5, clips=1, n=n, start=9)
    for amax, hop, want in ((600.0, 32, "umma"), (1024.0, 32, "umma"), (1024.0, 64, "umma"), (1024.0, 16, "umma"),
                            (1024.0, 128, "simt"), (1400.0, 32, "simt")):
        sc = np.geomspace(amax / 4, amax, 4)
        plan = wh.CwthPlan(sc, None, hop, n, wavelet="cmor", output="abs", max_clips=1, engine="auto")
        assert plan.engine == want, (amax, hop)
        got = plan.execute_host(x)
        plan.close()
        ref = O.cwth_batch(x, sc, hop, wavelet="cmor", output="abs")
        assert row_rel_err(got, ref) <= ROW_TOL, (amax, hop)
    with pytest.raises(Exception):
        wh.CwthPlan(np.geomspace(350.0, 1400.0, 4), None, 32, n, wavelet="cmor", output="abs", max_clips=1,
                    engine="umma")
    # min-max on a long-filter plan (the separate pass) and a real wavelet
    sc = np.geomspace(256.0, 1024.0, 3)
    plan = wh.CwthPlan(sc, None, 32, n, wavelet="rmor", output="abs", norm="minmax", max_clips=1, engine="umma")
    got = plan.execute_host(x)
    plan.close()
    ref = O.cwth_batch(x, sc, 32, wavelet="rmor", output="abs", norm="minmax")
    check_minmax(got, ref, O.cwth_batch(x, sc, 32, wavelet="rmor", output="abs"), "abs")


@pytest.mark.parametrize("hop,n", [(640, 1000), (640, 3000), (320, 5000), (1024, 20000)])
def test_panel_streaming_short_filters_and_short_clips(hop, n, monkeypatch):
    """Panel streaming with filters much shorter than a row of hop samples and clips of a few
    rows: the window origin falls inside a row, so a 64-sample panel must not straddle two
    rows of the batch tensor the TMA copies read (the K origin is a multiple of 64), the
    tensor has one or a few whole rows and the clip's partial last row comes from global memory."""
    monkeypatch.setenv("WH_UMMA_PSTREAM", "1")
    rng = np.random.default_rng(5)
    x = rng.standard_normal((2, n)).astype(np.float32)
    sc = np.geomspace(0.876, 51.487, 14)
    for wavelet, output in (("cmor", "power"), ("rmor", "abs")):
        plan = wh.CwthPlan(sc, None, hop, n, wavelet=wavelet, output=output, max_clips=2, engine="umma")
        got = plan.execute_host(x)
        # rows that are not 16-byte aligned: cp.async / scalar fetch and the scalar window scan
        base = np.zeros((2, n + 7), np.float32)
        base[:, 3:3 + n] = x
        got_u = plan.execute(torch.from_numpy(base).cuda()[:, 3:3 + n]).cpu().numpy()
        plan.close()
        ref = O.cwth_batch(x, sc, hop, wavelet=wavelet, output=output)
        assert got.shape == ref.shape
        tol = 2e-5 if output == "power" else ROW_TOL
        assert row_rel_err(got, ref) <= tol, (hop, n, wavelet)
        assert row_rel_err(got_u, ref) <= tol, (hop, n, wavelet, "unaligned")


@pytest.mark.parametrize("hop", [1280, 1344, 2048])
def test_panel_streaming_single_cta_units(hop):
    """Many clips of at most 128 frames at a large hop: a CTA pair's second tile would be empty,
    so the planner runs panel streaming with single-CTA MMAs (a unit = one 128-frame tile) --
    against the oracle, a NaN clip included."""
    n, clips = 24000, 200
    x = synth.make_batch(4, clips=clips, n=n, start=3)
    x[5, 7777] = np.nan
    sc = synth.config_scales(4)[::2]
    plan = wh.CwthPlan(sc, None, hop, n, wavelet="rmor", output="abs", max_clips=clips, engine="umma")
    got = plan.execute_host(x)
    plan.close()
    keep = np.array([i for i in range(clips) if i != 5])
    ref = O.cwth_batch(x[keep], sc, hop, wavelet="rmor", output="abs")
    assert got.shape == (clips, len(sc), -(-n // hop))
    assert row_rel_err(got[keep], ref) <= ROW_TOL
    k = np.arange(got.shape[2])
    for s_, a in enumerate(sc):
        L = math.ceil(6.0 * a * math.sqrt(0.75))
        np.testing.assert_array_equal(~np.isfinite(got[5, s_]), np.abs(k * hop - 7777) <= L)


@pytest.mark.parametrize("groups", ["2", "3", "8", "32"])
def test_pass_groups_are_byte_identical(groups, monkeypatch):
    """Splitting a tile pair's passes into separate units (what the launcher does when there
    are fewer tile pairs than CTA pairs, e.g. c3) changes only which CTA computes a pass:
    the outputs are byte-identical to the unsplit launch (hop 1: 32 passes; c5-like cmor
    min-max: 5 passes, the per-clip min / max then combines partial units)."""
    for cid, hop, wavelet, output, norm, clips, n in ((3, 1, "rmor", "abs", None, 2, 20000),
                                                      (5, 32, "cmor", "abs", "minmax", 3, 40000)):
        x = synth.make_batch(cid, clips=clips, n=n, start=1)
        sc = synth.config_scales(cid)
        plan = wh.CwthPlan(sc, None, hop, n, wavelet=wavelet, output=output, norm=norm,
                           max_clips=clips, engine="umma")
        monkeypatch.setenv("WH_UMMA_PGROUPS", "1")
        one = plan.execute_host(x).copy()
        monkeypatch.setenv("WH_UMMA_PGROUPS", groups)
        split = plan.execute_host(x)
        plan.close()
        assert one.tobytes() == split.tobytes(), (cid, groups)


@pytest.mark.parametrize("hop", [3, 6, 12, 24, 48, 96, 192])
def test_hops_dividing_192_on_tensor_cores(hop):
    """Hops whose rows are 192 samples (lcm(hop, 64) = 192: three 64-sample panels per row,
    P = 192/hop frames per row) run on the tensor-core engine and match the oracle; hop 192
    itself was accepted by the planner before row chunking handled non-power-of-two panels."""
    x = synth.make_batch(2, clips=2, n=20000, start=2)
    sc = synth.config_scales(2)
    plan = wh.CwthPlan(sc, None, hop, 20000, wavelet="rmor", output="abs", max_clips=2, engine="auto")
    assert plan.engine == "umma"
    got = plan.execute_host(x)
    plan.close()
    ref = O.cwth_batch(x, sc, hop, wavelet="rmor", output="abs")
    assert got.shape == (2, len(sc), -(-20000 // hop))
    assert row_rel_err(got, ref) <= ROW_TOL


@pytest.mark.parametrize("engine", ["umma", "simt"])
def test_unaligned_rows_and_odd_lengths(engine):
    """ld_x not a multiple of 4 (no 16-byte vector loads) and N not a multiple of the hop:
    same values as the packed layout."""
    rng = np.random.default_rng(21)
    n, ld = 10001, 10004 + 3
    base = rng.standard_normal((3, ld)).astype(np.float32)
    sc = np.geomspace(1.0, 40.0, 12)
    plan = wh.CwthPlan(sc, None, 16, n, wavelet="cmor", output="complex", max_clips=3, engine=engine)
    xt = torch.from_numpy(base).cuda()[:, 1:1 + n]  # offset view: rows not 16-byte aligned
    got = plan.execute(xt).cpu().numpy()
    ref = O.cwth_batch(base[:, 1:1 + n], sc, 16, output="complex")
    assert got.shape == ref.shape == (3, 12, -(-n // 16))
    assert row_rel_err(got, ref) <= ROW_TOL


def test_long_signal_and_empty_batch():
    """A 5M-sample clip (sample offsets far beyond 2^16 tiles of rows) and a zero-clip call."""
    rng = np.random.default_rng(33)
    n = 5_000_000
    x = rng.standard_normal((1, n)).astype(np.float32)
    sc = [1.0, 3.0, 9.0, 27.0]
    for hop, engine in ((64, "umma"), (1024, "umma"), (7, "simt")):
        got = wh.cwth_batch(x, sc, None, hop, wavelet="cmor", output="abs", engine=engine)
        ref = O.cwth_batch(x, sc, hop, wavelet="cmor", output="abs")
        assert got.shape == ref.shape == (1, 4, -(-n // hop))
        assert row_rel_err(got, ref) <= ROW_TOL, (hop, engine)
    plan = wh.CwthPlan(sc, None, 64, 1000, max_clips=2)
    empty = plan.execute(torch.empty((0, 1000), dtype=torch.float32, device="cuda"))
    assert tuple(empty.shape) == (0, 4, 16)


@pytest.mark.parametrize("engine", ENGINES)
def test_plans_sharing_a_kernel_keep_their_shared_memory(engine):
    """A plan created after another one with the same kernel instantiation but a smaller
    shared-memory footprint must not break the earlier plan's launches (the kernel's dynamic
    smem attribute is per function, not per plan)."""
    x = synth.make_batch(2, clips=2, n=20000)
    big = wh.CwthPlan(np.geomspace(1, 128, 16), None, 64, 20000, wavelet="rmor", output="abs", engine=engine,
                     max_clips=2)
    small = wh.CwthPlan(np.geomspace(1, 8, 16), None, 64, 20000, wavelet="rmor", output="abs", engine=engine,
                       max_clips=2)
    a = small.execute_host(x)
    b = big.execute_host(x)
    ref = O.cwth_batch(x, np.geomspace(1, 128, 16), 64, wavelet="rmor", output="abs")
    assert row_rel_err(b, ref) <= ROW_TOL and np.isfinite(a).all()
    big.close()
    small.close()


@pytest.mark.parametrize("mode", ["concurrent", "inkernel"])
def test_minmax_modes_byte_identical(mode, monkeypatch):
    """Per-clip min-max computed by the concurrent normaliser CTAs (beside k_umma, fed by the
    per-clip unit arrivals; WH_UMMA_MINMAX=concurrent) or in-kernel (=inkernel) gives the
    separate pass's bytes -- the concurrent one also for a clip with a non-finite sample (left
    to the trailing pass after the fix-up) -- over repeated launches of one plan."""
    x = synth.make_batch(5, clips=40, n=50000, start=11)
    if mode == "concurrent":  # (the in-kernel variant does not take non-finite input)
        x[7, 1234] = np.inf
    sc = synth.config_scales(5)
    mk = lambda: wh.CwthPlan(sc, None, 32, 50000, wavelet="cmor", output="abs", norm="minmax",  # noqa: E731
                             max_clips=40, engine="umma")
    plan = mk()
    want = plan.execute_host(x).copy()
    plan.close()
    monkeypatch.setenv("WH_UMMA_MINMAX", mode)
    plan = mk()
    xd = torch.from_numpy(x).cuda()
    for _ in range(3):
        got = plan.execute(xd).cpu().numpy()
        assert got.tobytes() == want.tobytes()
    plan.close()


def test_cached_plan_survives_eviction():
    """get_plan's LRU eviction (and replacement by a larger plan) drops the cache's reference
    only: a caller still holding the plan keeps a working plan (closed when the last reference
    goes), instead of one freed under it."""
    from paper_2408_14302_b200.wavelet import get_plan

    x = synth.make_batch(2, clips=1, n=8000)
    kw = dict(wavelet="rmor", output="abs", norm=None, clips=1, device=0, engine="auto")
    held = get_plan(np.geomspace(1, 16, 8), None, 16, 8000, **kw)
    first = held.execute_host(x).copy()
    for i in range(20):  # more than the cache holds
        get_plan(np.geomspace(1, 16, 8) * (1 + 0.01 * (i + 1)), None, 16, 8000, **kw)
    get_plan(np.geomspace(1, 16, 8), None, 16, 8000, **{**kw, "clips": 4})  # replaces the key
    np.testing.assert_array_equal(held.execute_host(x), first)
