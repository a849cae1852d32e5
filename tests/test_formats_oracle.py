"""SURVEY.md §8f rows (decimate, cwth_decimate, render, SCG1/PGM/CSV): the oracle
restatements and the product's host-side writers against golden vectors from the
unmodified reference (oracle/gen_golden.py -> tests/golden/formats.npz).  CPU only."""
import os

import numpy as np
import pytest

from conftest import decimate_cases, max_rel_err
from oracle import oracle as O
import paper_2408_14302_b200 as wh
from paper_2408_14302_b200 import scalogram as S


def test_firwin_restatement_matches_scipy():
    # the reference's dependency (signal_io.py:144), restated: same taps to rounding
    sig = pytest.importorskip("scipy.signal")
    for hop in (1, 2, 4, 7, 16, 64, 128):
        ref = sig.firwin(10 * hop + 1, 0.9 / hop)
        got = O.firwin_lowpass(10 * hop + 1, 0.9 / hop)
        assert np.abs(got - ref).max() <= 1e-15


def test_decimate_matches_reference(golden_formats):
    cases = decimate_cases(golden_formats, "d_")
    assert len(cases) == 7
    for name, c in cases:
        hop, aa = (int(v) for v in c["meta"])
        got = O.decimate(c["x"].astype(np.float64), hop, bool(aa))
        assert got.shape == c["ref"].shape == (-(-c["x"].size // hop),), name
        if aa:
            assert max_rel_err(got, c["ref"]) <= 1e-12, name  # fftconvolve vs direct sum
        else:
            np.testing.assert_array_equal(got, c["ref"])  # pure selection: bit-exact
        assert float(c["rate"]) == 16000.0 / hop


def test_cwth_decimate_matches_reference(golden_formats):
    cases = decimate_cases(golden_formats, "cd_")
    assert len(cases) == 3
    for name, c in cases:
        hop, aa, mhop = (int(v) for v in c["meta"])
        assert mhop == hop and float(c["rate"]) == 16000.0 / hop
        got = O.cwth_decimate_batch(c["x"][None].astype(np.float64), c["scales"], hop, bool(aa))[0]
        assert got.shape == c["ref"].shape
        assert max_rel_err(got, c["ref"]) <= 1e-9, name  # reference: FFT rows


def test_render_restatement_exact(golden_formats):
    g = golden_formats
    v = g["render_rand__v"].astype(np.float64)
    np.testing.assert_array_equal(O.render(v), g["render_rand__flip"])
    np.testing.assert_array_equal(O.render(v, flip_vertical=False), g["render_rand__noflip"])
    np.testing.assert_array_equal(O.render(g["render_ties__v"]), g["render_ties__flip"])
    np.testing.assert_array_equal(O.render(g["render_const__v"]), g["render_const__flip"])
    assert g["render_const__flip"].max() == 0


def test_scg1_bytes_and_writers_byte_exact(golden_formats, golden_cwth, tmp_path):
    g = golden_formats
    vals = golden_cwth["c5s__ref"]
    scales = np.geomspace(1, 512, 12)
    ref_bin = g["file_scg1"].tobytes()
    assert O.scg1_bytes(vals, 32, 16000.0, scales) == ref_bin
    # the product's writers (host code, no device needed)
    m = wh.CoefficientMatrix(vals, 32, 16000.0, wh.ScaleGrid(scales))
    S.write_matrix_bin(m, tmp_path / "m.scg1")
    assert (tmp_path / "m.scg1").read_bytes() == ref_bin
    S.write_matrix_bin_raw(vals.astype(np.complex64), 32, 16000.0, scales, tmp_path / "r.scg1")
    assert (tmp_path / "r.scg1").read_bytes() == ref_bin
    back = S.read_matrix_bin(tmp_path / "m.scg1")
    assert back.hop == 32 and back.source_rate == 16000.0
    np.testing.assert_array_equal(back.values, vals.astype(np.complex64).astype(np.complex128))
    np.testing.assert_array_equal(back.scale_grid.scales, scales)
    img = S.ScalogramImage(O.render(np.abs(vals)))
    S.write_pgm(img, tmp_path / "m.pgm")
    assert (tmp_path / "m.pgm").read_bytes() == g["file_pgm"].tobytes()
    S.write_csv(S.magnitude(m, "log_db")[:3, :10], tmp_path / "m.csv")
    assert (tmp_path / "m.csv").read_bytes() == g["file_csv"].tobytes()


def test_read_matrix_bin_errors(tmp_path):
    p = tmp_path / "bad.scg1"
    p.write_bytes(b"XXXX")
    with pytest.raises(wh.MalformedHeader):
        S.read_matrix_bin(p)
    p.write_bytes(b"SCG1" + b"\x00" * 8)
    with pytest.raises(wh.MalformedHeader):
        S.read_matrix_bin(p)
    blob = O.scg1_bytes(np.ones((2, 3), np.complex64), 4, 8000.0, [1.0, 2.0])
    p.write_bytes(blob[:-5])
    with pytest.raises(wh.TruncatedPayload):
        S.read_matrix_bin(p)
    with pytest.raises(wh.IoFailure):
        S.read_matrix_bin(tmp_path / "missing.scg1")


def test_wav_codec_matches_reference(golden_formats, tmp_path):
    """WAV files written and read by the reference (signal_io.py:165-250) are byte-identical /
    decode identically (pcm16, float32, a stereo file averaged to mono, malformed input)."""
    from paper_2408_14302_b200 import wavio

    g = golden_formats
    sig = wh.SignalBuffer(np.sin(np.arange(300) * 0.05) * 0.9, 11025.0)
    for enc in ("pcm16", "float32"):
        wavio.write_wav(sig, tmp_path / f"{enc}.wav", encoding=enc)
        assert (tmp_path / f"{enc}.wav").read_bytes() == g[f"wav_{enc}"].tobytes()
        np.testing.assert_array_equal(wavio.read_wav(tmp_path / f"{enc}.wav").samples, g[f"wav_{enc}__read"])
    (tmp_path / "st.wav").write_bytes(g["wav_stereo"].tobytes())
    st = wavio.read_wav(tmp_path / "st.wav")
    np.testing.assert_array_equal(st.samples, g["wav_stereo__read"])
    assert st.sample_rate == 22050.0
    (tmp_path / "bad.wav").write_bytes(b"RIFF\x00\x00\x00\x00WAVX")
    with pytest.raises(wh.MalformedRiff):
        wavio.read_wav(tmp_path / "bad.wav")
    blob = bytearray(g["wav_pcm16"].tobytes())
    blob[22:24] = (2).to_bytes(2, "little")  # claim 2 channels: 300 samples -> 150 frames
    (tmp_path / "two.wav").write_bytes(bytes(blob))
    assert wavio.read_wav(tmp_path / "two.wav").samples.size == 150
    blob = bytearray(g["wav_pcm16"].tobytes())
    blob[20:22] = (3).to_bytes(2, "little")  # IEEE float tag with 16 bits
    (tmp_path / "enc.wav").write_bytes(bytes(blob))
    with pytest.raises(wh.UnsupportedEncoding):
        wavio.read_wav(tmp_path / "enc.wav")
    with pytest.raises(wh.IoFailure):
        wavio.read_wav(tmp_path / "missing.wav")


def test_cli_parsing_and_errors(tmp_path, capsys):
    from paper_2408_14302_b200 import cli

    assert cli.run_cli([]) == 2  # usage error
    assert cli.run_cli(["scan", str(tmp_path), "--out-dir", str(tmp_path / "o")]) == 1
    assert "no .wav files" in capsys.readouterr().err
    assert cli.run_cli(["transform", str(tmp_path / "missing.wav"), "--out", str(tmp_path / "m.scg1")]) == 1
    assert cli.run_cli(["scalogram", str(tmp_path / "missing.scg1"), "--out", str(tmp_path / "x.pgm")]) == 1
