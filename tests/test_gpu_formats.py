"""SURVEY.md §8f rows on the GPU through the C ABI: decimation (wh_decimate), cwth_decimate
(decimate + hop-1 plan), render (wh_render_u8 and the fused WH_NORM_RENDER_U8 plans) and
the SCG1 payload written straight from the device result -- against the oracle and the
reference's golden vectors (tests/golden/formats.npz)."""
import numpy as np
import pytest
import torch

from conftest import decimate_cases, max_rel_err, row_rel_err
from oracle import oracle as O
import paper_2408_14302_b200 as wh
from paper_2408_14302_b200 import scalogram as S
from paper_2408_14302_b200 import synth

pytestmark = pytest.mark.gpu


def test_decimate_device_matches_reference(golden_formats):
    for name, c in decimate_cases(golden_formats, "d_"):
        hop, aa = (int(v) for v in c["meta"])
        got = wh.decimate_device(torch.from_numpy(c["x"]).cuda(), hop, bool(aa)).cpu().numpy()
        assert got.shape == c["ref"].shape, name
        if aa:  # float64 accumulation, float32 result
            assert max_rel_err(got, c["ref"]) <= 1e-6, name
        else:
            np.testing.assert_array_equal(got, c["ref"].astype(np.float32))
        sig = wh.decimate(wh.SignalBuffer(c["x"].astype(np.float64), 16000.0), hop, bool(aa))
        assert sig.sample_rate == float(c["rate"]) and sig.samples.shape == c["ref"].shape


def test_decimate_batch_ragged_and_errors():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((3, 1001)).astype(np.float32)
    for hop in (1, 3, 16, 1000, 2000):
        got = wh.decimate_device(torch.from_numpy(x).cuda(), hop, True).cpu().numpy()
        ref = O.decimate(x.astype(np.float64), hop, True)
        assert got.shape == ref.shape == (3, -(-1001 // hop))
        assert max_rel_err(got, ref) <= 1e-6
    with pytest.raises(wh.InvalidHop):
        wh.decimate_device(torch.from_numpy(x).cuda(), 0)


def test_cwth_decimate_matches_reference(golden_formats):
    for name, c in decimate_cases(golden_formats, "cd_"):
        hop, aa, _ = (int(v) for v in c["meta"])
        m = wh.cwth_decimate(wh.SignalBuffer(c["x"].astype(np.float64), 16000.0),
                             wh.ScaleGrid(c["scales"]), None, hop, bool(aa))
        assert m.hop == hop and m.source_rate == float(c["rate"])
        assert m.values.shape == c["ref"].shape
        assert row_rel_err(m.values, c["ref"]) <= 1e-5, name


def test_cwth_decimate_batch_full_size():
    """c2-sized clips decimated by 64 (anti-aliased), log1p of |Re W| at hop 1 on 2,500
    samples, against the float64 oracle."""
    x = synth.make_batch(2, clips=3, start=7)
    sc = np.geomspace(1.0, 32.0, 24)
    got = wh.cwth_decimate_batch(x, sc, None, 64, True, wavelet="rmor", output="log1p")
    ref = O.cwth_decimate_batch(x, sc, 64, True, wavelet="rmor", output="log1p")
    assert got.shape == ref.shape == (3, 24, 2500)
    assert np.abs(got - ref).max() <= 1e-5


def test_render_device_matches_reference(golden_formats):
    g = golden_formats
    for key, flip in (("render_rand__flip", True), ("render_rand__noflip", False)):
        got = S.render(g["render_rand__v"], flip_vertical=flip).pixels
        np.testing.assert_array_equal(got, g[key])
    np.testing.assert_array_equal(S.render(g["render_ties__v"]).pixels, g["render_ties__flip"])
    np.testing.assert_array_equal(S.render(g["render_const__v"]).pixels, g["render_const__flip"])
    # batched: each matrix normalised on its own
    v = torch.from_numpy(np.stack([g["render_rand__v"], 3.0 * g["render_rand__v"] + 1])).cuda()
    px = S.render_device(v).cpu().numpy()
    np.testing.assert_array_equal(px[0], g["render_rand__flip"])
    np.testing.assert_array_equal(px[1], O.render(3.0 * g["render_rand__v"].astype(np.float32) + 1))


@pytest.mark.parametrize("norm,flip", [("render", True), ("render_noflip", False)])
def test_fused_render_plan(norm, flip):
    """norm="render": the plan's fp32 magnitudes mapped to uint8 per clip -- byte-exact
    against render() of the same plan's float output, within one level of the float64
    oracle."""
    x = synth.make_batch(5, clips=3, n=40000, start=2)
    sc = synth.config_scales(5)
    for output in ("abs", "log_db"):
        px = wh.cwth_batch(x, sc, None, 32, wavelet="cmor", output=output, norm=norm)
        vals = wh.cwth_batch(x, sc, None, 32, wavelet="cmor", output=output)
        assert px.dtype == np.uint8 and px.shape == vals.shape
        for c in range(3):
            np.testing.assert_array_equal(px[c], O.render(vals[c], flip_vertical=flip))
            ref = O.render(O.cwth_batch(x[c:c + 1], sc, 32, wavelet="cmor", output=output)[0],
                           flip_vertical=flip)
            assert np.abs(px[c].astype(int) - ref.astype(int)).max() <= 1


def test_fused_render_host_path_and_constant_clip():
    x = np.zeros((2, 5000), np.float32)
    x[1, 100] = 1.0
    plan = wh.CwthPlan([2.0, 8.0], None, 16, 5000, wavelet="cmor", output="abs", norm="render",
                       max_clips=2)
    host = plan.execute_host(x)
    dev = plan.execute(torch.from_numpy(x).cuda()).cpu().numpy()
    np.testing.assert_array_equal(host, dev)
    assert host[0].max() == 0  # constant clip -> zeros (scalogram.py:79-80)
    assert host[1].max() == 255


def test_scg1_from_device_payload(tmp_path):
    """The device complex64 layout is the SCG1 payload: write it without conversion and
    read it back through the reference-format reader."""
    x = synth.make_batch(1, clips=1)
    sc = synth.config_scales(1)
    vals = wh.cwth_batch(x, sc, None, 16, wavelet="cmor", output="complex")[0]
    S.write_matrix_bin_raw(vals, 16, 16000.0, sc, tmp_path / "a.scg1")
    assert (tmp_path / "a.scg1").read_bytes() == O.scg1_bytes(vals, 16, 16000.0, sc)
    back = S.read_matrix_bin(tmp_path / "a.scg1")
    np.testing.assert_array_equal(back.values, vals.astype(np.complex128))
