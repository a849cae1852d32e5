"""The reference's own tests for the §8f rows (pkg/tests/test_cli.py, test_bench.py,
test_scalogram.py TestRender, test_signal_io.py TestDecimate), restated against the GPU
path of this package.  Deviations: ``bench_single(include_dwt=True)`` raises (the DWT is not
on the GPU path); the ``auc`` subcommand does not exist."""
import json
import math

import numpy as np
import pytest

import paper_2408_14302_b200 as wh
from paper_2408_14302_b200 import cli, scalogram as S, wavio
import signals
from paper_2408_14302_b200.bench import BenchReport, bench_single, extrapolate_dataset, reports_to_jsonl

pytestmark = pytest.mark.gpu
PARAMS = wh.MorletParams()
run_cli = cli.run_cli


def make_wav(path, n=4000, seed=0, rate=16_000.0):
    x = np.random.default_rng(seed).uniform(-0.8, 0.8, n)
    wavio.write_wav(wh.SignalBuffer(x, rate), path)


# ---- test_signal_io.py TestDecimate -------------------------------------------------------

def test_decimate_plain_index_selection():
    out = wh.decimate(wh.SignalBuffer([0, 1, 2, 3, 4, 5], 16_000), 2)
    np.testing.assert_array_equal(out.samples, [0, 2, 4])
    assert out.sample_rate == 8000


def test_decimate_hop_one_is_identity():
    sig = wh.SignalBuffer(np.random.default_rng(0).standard_normal(999), 44_100, "x")
    out = wh.decimate(sig, 1)
    np.testing.assert_array_equal(out.samples, sig.samples)
    assert out.sample_rate == sig.sample_rate and out.source_label == sig.source_label


@pytest.mark.parametrize("n,hop", [(10, 3), (11, 3), (12, 3), (1, 5), (100, 7), (160_000, 128)])
def test_decimate_ceil_length(n, hop):
    assert len(wh.decimate(wh.SignalBuffer(np.arange(n, dtype=float), 8000), hop)) == math.ceil(n / hop)


def test_decimate_composition_and_invalid_hop():
    sig = wh.SignalBuffer(np.random.default_rng(1).standard_normal(1000).astype(np.float32), 16_000)
    nested = wh.decimate(wh.decimate(sig, 3), 4)
    flat = wh.decimate(sig, 12)
    np.testing.assert_array_equal(nested.samples, flat.samples)
    assert math.isclose(nested.sample_rate, flat.sample_rate, rel_tol=1e-12)
    with pytest.raises(wh.InvalidHop):
        wh.decimate(wh.SignalBuffer([1.0, 2.0], 8000), 0)


def test_anti_alias_suppresses_folding_and_passes_low_frequencies():
    hi = signals.sine(8000, 16_000, 3600.0)
    plain, filt = wh.decimate(hi, 4).samples, wh.decimate(hi, 4, anti_alias=True).samples
    assert len(filt) == len(plain)
    assert np.sqrt(np.mean(filt ** 2)) < 0.05 * np.sqrt(np.mean(plain ** 2))
    lo = signals.sine(8000, 16_000, 200.0)
    plain, filt = wh.decimate(lo, 4).samples, wh.decimate(lo, 4, anti_alias=True).samples
    assert np.max(np.abs(filt[100:-100] - plain[100:-100])) < 0.02


# ---- test_scalogram.py TestRender (on the GPU) --------------------------------------------

def test_render_reference_cases():
    assert np.all(S.render(np.full((3, 4), 2.5)).pixels == 0)
    assert S.render(np.array([[0.0, 1.0]]), flip_vertical=False).pixels.tolist() == [[0, 255]]
    assert S.render(np.array([[0.0, 0.5, 1.0]]), flip_vertical=False).pixels.tolist() == [[0, 128, 255]]
    values = np.array([[0.0, 0.0], [1.0, 1.0]])
    assert S.render(values, flip_vertical=False).pixels[0].tolist() == [0, 0]
    assert S.render(values, flip_vertical=True).pixels[0].tolist() == [255, 255]
    img = S.render(np.random.default_rng(1).standard_normal((6, 40)))
    assert img.pixels.min() == 0 and img.pixels.max() == 255
    with pytest.raises(ValueError):
        S.render(np.zeros((0, 3)))


# ---- test_bench.py ------------------------------------------------------------------------

def small_workload():
    sig = signals.white_noise(8192, 16_000.0, seed=3)
    return sig, wh.make_scale_grid(300.0, 3000.0, 8, 16_000.0, PARAMS)


def test_bench_reports_shape_and_reference():
    signal, grid = small_workload()
    reports = bench_single(signal, grid, PARAMS, hop=64, reps=3)
    by = {r.method: r for r in reports}
    assert set(by) == {"cwt_fft", "cwth_strided"}
    assert by["cwt_fft"].speedup_vs_full == 1.0 and by["cwt_fft"].hop == 1
    for r in reports:
        assert r.signal_length == 8192 and r.scale_count == 8 and r.repetitions == 3
        assert r.median_seconds > 0 and r.min_seconds <= r.median_seconds and r.speedup_vs_full > 0
    assert by["cwth_strided"].hop == 64
    methods = [r.method for r in bench_single(signal, grid, PARAMS, hop=64, reps=3, include_decimate=True)]
    assert methods == ["cwt_fft", "cwth_strided", "cwth_decimate"]
    with pytest.raises(ValueError):
        bench_single(signal, grid, PARAMS, hop=64, reps=2)
    with pytest.raises(ValueError):  # documented deviation: no DWT on the GPU path
        bench_single(signal, grid, PARAMS, hop=64, reps=3, include_dwt=True)


def test_bench_timing_does_not_perturb_results():
    signal, grid = small_workload()
    before = wh.cwth_strided(signal, grid, PARAMS, 64).values
    bench_single(signal, grid, PARAMS, hop=64, reps=3)
    np.testing.assert_array_equal(before, wh.cwth_strided(signal, grid, PARAMS, 64).values)


def test_bench_json_and_extrapolation():
    report = BenchReport("cwt_fft", 100, 4, 1, 3, 0.5, 0.4, 1.0)
    assert list(json.loads(report.to_json())) == ["method", "signal_length", "scale_count", "hop",
                                                  "repetitions", "median_seconds", "min_seconds",
                                                  "speedup_vs_full"]
    signal, grid = small_workload()
    reports = bench_single(signal, grid, PARAMS, hop=32, reps=3)
    lines = reports_to_jsonl(reports).strip().split("\n")
    assert [json.loads(l)["method"] for l in lines] == [r.method for r in reports]
    r = BenchReport("cwth_strided", 160_000, 64, 128, 5, 0.15, 0.14, 50.0)
    assert extrapolate_dataset(r, 54_507) == pytest.approx(0.15 * 54_507 / 3600.0, rel=1e-15)
    assert extrapolate_dataset(report, 1) == 0.5 / 3600.0
    with pytest.raises(ValueError):
        extrapolate_dataset(report, 0)


# ---- test_cli.py ---------------------------------------------------------------------------

def wav_of(tmp_path, name, sig):
    path = tmp_path / name
    wavio.write_wav(sig, path, encoding="float32")
    return str(path)


def test_transform_commands(tmp_path, capsys):
    wav = tmp_path / "in.wav"
    make_wav(wav, n=160_000)
    out = tmp_path / "out.scg1"
    assert run_cli(["transform", str(wav), "--out", str(out), "--mode", "strided", "--hop", "128",
                    "--scales", "8", "--fmin", "500", "--fmax", "4000"]) == 0
    m = S.read_matrix_bin(out)
    assert (m.columns, m.hop, m.rows) == (1250, 128, 8)
    sine = wav_of(tmp_path, "sine.wav", signals.sine(4096, 16_000, 1000.0, 0.5))
    assert run_cli(["transform", sine, "--out", str(out), "--hop", "64", "--scales", "6", "--fmin", "500",
                    "--fmax", "4000"]) == 0
    assert S.read_matrix_bin(out).columns == 64
    n1 = wav_of(tmp_path, "n1.wav", signals.white_noise(16000, 16_000, 1))
    assert run_cli(["transform", n1, "--out", str(out), "--mode", "decimate", "--hop", "4", "--scales", "6",
                    "--fmin", "100", "--fmax", "1500"]) == 0
    m = S.read_matrix_bin(out)
    assert (m.source_rate, m.hop, m.columns) == (4000.0, 4, 4000)
    n2 = wav_of(tmp_path, "n2.wav", signals.white_noise(2048, 16_000, 2))
    assert run_cli(["transform", n2, "--out", str(out), "--mode", "full", "--scales", "4", "--fmin", "500",
                    "--fmax", "4000"]) == 0
    m = S.read_matrix_bin(out)
    assert (m.columns, m.hop) == (2048, 1)
    csv, pgm = tmp_path / "o.csv", tmp_path / "o.pgm"
    n4 = wav_of(tmp_path, "n4.wav", signals.white_noise(2000, 16_000, 4))
    assert run_cli(["transform", n4, "--out", str(out), "--csv", str(csv), "--pgm", str(pgm), "--hop", "50",
                    "--scales", "5", "--fmin", "500", "--fmax", "4000", "--mag", "log_db"]) == 0
    assert csv.read_text().count("\n") == 5
    assert pgm.read_bytes().startswith(b"P5\n40 5\n255\n")
    assert run_cli(["transform", str(tmp_path / "none.wav"), "--out", str(tmp_path / "x.scg1")]) == 1
    assert "error" in capsys.readouterr().err


def test_transform_byte_deterministic(tmp_path):
    n5 = wav_of(tmp_path, "n5.wav", signals.white_noise(3000, 16_000, 5))
    args = ["transform", n5, "--mode", "strided", "--hop", "30", "--scales", "6", "--fmin", "300",
            "--fmax", "3000"]
    outs = []
    for tag in ("a", "b"):
        o, p = tmp_path / f"{tag}.scg1", tmp_path / f"{tag}.pgm"
        assert run_cli(args + ["--out", str(o), "--pgm", str(p)]) == 0
        outs.append((o.read_bytes(), p.read_bytes()))
    assert outs[0] == outs[1]


def test_scalogram_command_and_flip(tmp_path):
    out = tmp_path / "o.scg1"
    t = np.arange(4000) / 16_000.0
    chirp = wh.SignalBuffer(np.sin(2 * np.pi * (200.0 * t + 0.5 * (3800.0 / t[-1]) * t * t)), 16_000.0)
    src = wav_of(tmp_path, "chirp.wav", chirp)
    run_cli(["transform", src, "--out", str(out), "--hop", "40", "--scales", "6", "--fmin", "300",
             "--fmax", "3000"])
    a, b = tmp_path / "a.pgm", tmp_path / "b.pgm"
    assert run_cli(["scalogram", str(out), "--out", str(a)]) == 0
    assert a.read_bytes().startswith(b"P5\n100 6\n255\n")
    run_cli(["scalogram", str(out), "--out", str(b), "--no-flip"])
    assert a.read_bytes() != b.read_bytes()


def test_usage_errors(capsys):
    assert run_cli(["transform", "x.wav", "--out", "x.scg1", "--bogus"]) == 2
    assert "usage" in capsys.readouterr().err.lower()
    assert run_cli([]) == 2
    assert run_cli(["fourier"]) == 2


def test_bench_command(capsys):
    assert run_cli(["bench", "--length", "8192", "--rate", "16000", "--hop", "64", "--reps", "3",
                    "--scales", "6", "--fmin", "300", "--fmax", "3000"]) == 0
    decoded = [json.loads(l) for l in capsys.readouterr().out.strip().split("\n")]
    assert [d["method"] for d in decoded] == ["cwt_fft", "cwth_strided"]
    assert all(d["signal_length"] == 8192 for d in decoded)


def test_scan_command_reference_cases(tmp_path, capsys, monkeypatch):
    base = ["--hop", "40", "--scales", "5", "--fmin", "300", "--fmax", "3000"]
    in_dir = tmp_path / "in"
    in_dir.mkdir()
    for name, seed in (("b.wav", 1), ("a.wav", 2), ("c.wav", 3)):
        make_wav(in_dir / name, n=4000, seed=seed)
    out_dir = tmp_path / "out"
    assert run_cli(["scan", str(in_dir), "--out-dir", str(out_dir)] + base) == 0
    assert sorted(p.name for p in out_dir.iterdir()) == ["a.scg1", "b.scg1", "c.scg1"]
    assert capsys.readouterr().out.strip().split("\n") == ["ok a.wav", "ok b.wav", "ok c.wav"]
    (in_dir / "bad.wav").write_bytes(b"not a wav at all")
    out2 = tmp_path / "out2"
    assert run_cli(["scan", str(in_dir), "--out-dir", str(out2)] + base) == 1
    assert (out2 / "a.scg1").exists() and not (out2 / "bad.scg1").exists()
    cap = capsys.readouterr()
    assert "ok a.wav" in cap.out and "failed bad.wav" in cap.err
    # threads give identical bytes; THREADS env honoured
    (in_dir / "bad.wav").unlink()
    t1, t3 = tmp_path / "t1", tmp_path / "t3"
    assert run_cli(["scan", str(in_dir), "--out-dir", str(t1)] + base) == 0
    monkeypatch.setenv("THREADS", "3")
    assert run_cli(["scan", str(in_dir), "--out-dir", str(t3)] + base) == 0
    for p in sorted(t1.iterdir()):
        assert p.read_bytes() == (t3 / p.name).read_bytes()
    empty = tmp_path / "empty"
    empty.mkdir()
    assert run_cli(["scan", str(empty), "--out-dir", str(tmp_path / "o3")]) == 1
