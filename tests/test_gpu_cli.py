"""SURVEY.md §8f rows 1 and 3 on the GPU: the CLI's transform / scalogram / bench and the
batched ``scan`` driver, against the oracle and the single-file public API."""
import json

import numpy as np
import pytest

from conftest import row_rel_err
from oracle import oracle as O
import paper_2408_14302_b200 as wh
from paper_2408_14302_b200 import cli, scalogram as S, wavio
import signals

pytestmark = pytest.mark.gpu


def _grid(rate, n_scales=24, fmin=50.0, fmax=None):
    return wh.make_scale_grid(fmin, fmax or 0.45 * rate, n_scales, rate)


@pytest.mark.parametrize("mode", ["strided", "decimate", "full"])
def test_transform_command(tmp_path, mode):
    out = tmp_path / "a.scg1"
    sig = signals.white_noise(8000, 8000.0, seed=3)
    wavio.write_wav(sig, tmp_path / "in.wav", encoding="float32")
    argv = ["transform", str(tmp_path / "in.wav"), "--out", str(out),
            "--mode", mode, "--hop", "16", "--scales", "24", "--fmin", "50",
            "--csv", str(tmp_path / "a.csv"), "--pgm", str(tmp_path / "a.pgm")]
    if mode == "decimate":
        argv.append("--anti-alias")
    assert cli.run_cli(argv) == 0
    m = S.read_matrix_bin(out)
    sig = wavio.read_wav(tmp_path / "in.wav")  # float32 on disk: the samples the CLI saw
    rate = 8000.0 / 16 if mode == "decimate" else 8000.0
    grid = _grid(rate)
    np.testing.assert_array_equal(m.scale_grid.scales, grid.scales)
    if mode == "strided":
        ref = O.cwth_batch(sig.samples.astype(np.float32), grid.scales, 16)
        assert m.hop == 16 and m.source_rate == 8000.0
    elif mode == "full":
        ref = O.cwth_batch(sig.samples.astype(np.float32), grid.scales, 1)
        assert m.hop == 1
    else:
        ref = O.cwth_decimate_batch(sig.samples.astype(np.float32)[None], grid.scales, 16, True)[0]
        assert m.hop == 16 and m.source_rate == 500.0
    assert m.values.shape == ref.shape
    assert row_rel_err(m.values, ref) <= 1e-5
    assert (tmp_path / "a.pgm").read_bytes().startswith(f"P5\n{ref.shape[1]} {ref.shape[0]}\n255\n".encode())
    assert len((tmp_path / "a.csv").read_text().splitlines()) == ref.shape[0]
    # scalogram command re-renders the stored matrix
    assert cli.run_cli(["scalogram", str(out), "--out", str(tmp_path / "b.pgm"), "--no-flip"]) == 0
    px = np.frombuffer((tmp_path / "b.pgm").read_bytes()[-ref.size:], np.uint8).reshape(ref.shape)
    np.testing.assert_array_equal(px, O.render(np.abs(m.values).astype(np.float32), flip_vertical=False))


def test_bench_command_jsonl(capsys):
    assert cli.run_cli(["bench", "--length", "16000", "--hop", "64", "--reps", "3", "--scales", "16",
                        "--include-decimate"]) == 0
    lines = [json.loads(l) for l in capsys.readouterr().out.splitlines()]
    assert [r["method"] for r in lines] == ["cwt_fft", "cwth_strided", "cwth_decimate"]
    for r in lines:
        assert set(r) == {"method", "signal_length", "scale_count", "hop", "repetitions",
                          "median_seconds", "min_seconds", "speedup_vs_full"}
        assert r["signal_length"] == 16000 and r["scale_count"] == 16 and r["repetitions"] == 3
        assert r["median_seconds"] > 0 and r["min_seconds"] <= r["median_seconds"]
    assert lines[0]["speedup_vs_full"] == 1.0 and lines[1]["hop"] == 64 and lines[0]["hop"] == 1
    with pytest.raises(ValueError):
        wh.bench.bench_single(wh.SignalBuffer(np.ones(10), 8000.0), wh.ScaleGrid([1.0]), reps=2)


def test_scan_batched_matches_single_file(tmp_path, capsys):
    """scan groups equal-length files into one batched plan; each .scg1 is byte-identical to
    the single-file transform's SCG1 (per-clip work is identical), the PGMs within one
    level of render(magnitude(...)) of that matrix; a corrupt file fails alone."""
    src = tmp_path / "in"
    src.mkdir()
    rng = np.random.default_rng(11)
    for i in range(3):
        wavio.write_wav(wh.SignalBuffer(rng.uniform(-0.9, 0.9, 6000), 16000.0), src / f"a{i}.wav")
    wavio.write_wav(wh.SignalBuffer(rng.uniform(-0.9, 0.9, 4000), 16000.0), src / "b.wav", encoding="float32")
    (src / "c.wav").write_bytes(b"RIFF\x04\x00\x00\x00WAVE")
    out = tmp_path / "out"
    rc = cli.run_cli(["scan", str(src), "--out-dir", str(out), "--pgm", "--hop", "32", "--scales", "20", "--fmin", "50",
                      "--threads", "4"])
    cap = capsys.readouterr()
    assert rc == 1
    assert cap.out.splitlines() == ["ok a0.wav", "ok a1.wav", "ok a2.wav", "ok b.wav"]
    assert cap.err.startswith("failed c.wav: ")
    grid = _grid(16000.0, 20)
    for name in ("a0", "a1", "a2", "b"):
        sig = wavio.read_wav(src / f"{name}.wav")
        m = wh.cwth_strided(sig, grid, None, 32)
        S.write_matrix_bin(m, tmp_path / "single.scg1")
        assert (out / f"{name}.scg1").read_bytes() == (tmp_path / "single.scg1").read_bytes()
        pgm = (out / f"{name}.pgm").read_bytes()
        px = np.frombuffer(pgm[-m.values.size:], np.uint8).reshape(m.values.shape)
        ref = O.render(np.abs(m.values))
        assert np.abs(px.astype(int) - ref.astype(int)).max() <= 1
