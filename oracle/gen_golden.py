"""Generate tests/golden/*.npz from the UNMODIFIED reference package.

Run here (the reference is importable only in the build container):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden.py

It imports wavehop 0.1.0 read-only from /root/reference/pkg/src and records, for
seeded inputs, what the reference's own public API returns:

* ``taps.npz``   -- sample_wavelet (wavelet.py:144-159) for selected scales and the
                    half widths L (wavelet.py:154) of every scale in every BASELINE config;
* ``cwth.npz``   -- cwth_strided (wavelet.py:215-273) complex128 outputs for small
                    versions of c1-c5 plus ragged/edge/impulse/parameter cases, and
                    magnitude/render (scalogram.py:51-86) outputs;
* ``formats.npz`` -- the SURVEY §8f rows: decimate (signal_io.py:130-150, with and
                    without the anti-alias FIR), cwth_decimate (wavelet.py:276-294),
                    render on float32 matrices incl. exact .5 ties and a constant
                    matrix, and the bytes of write_matrix_bin / write_pgm / write_csv.

The GPU box never reads /root/reference; tests read only these fixtures.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import wavehop  # noqa: E402  (reference)
from wavehop import (MorletParams, ScaleGrid, SignalBuffer, SynthSpec, cwth_strided,  # noqa: E402
                     make_scale_grid, magnitude, render, sample_wavelet, synthesize)

from paper_2408_14302_b200 import synth  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")


def ref_cwth(x32, scales, hop, params=None):
    sig = SignalBuffer(np.asarray(x32, dtype=np.float32).astype(np.float64), 16_000.0)
    return cwth_strided(sig, ScaleGrid(np.asarray(scales, dtype=np.float64)), params, hop).values


def main():
    os.makedirs(OUT, exist_ok=True)
    params = MorletParams()

    # ---- taps -------------------------------------------------------------------------
    taps = {}
    for cid in synth.CONFIGS:
        sc = synth.config_scales(cid)
        taps[f"scales_c{cid}"] = sc
        taps[f"half_c{cid}"] = np.array(
            [sample_wavelet(params, s).size // 2 for s in sc], dtype=np.int64)
    pick = [1.0, 2.5, 4.0, 9.3, 12.0, 37.5, 80.0, 128.0, 511.99, 512.0]
    c5 = synth.config_scales(5)
    # the c5 scale whose R*a*sqrt(B/2) lands closest to an integer (SURVEY.md §7 hard parts)
    prod = 6.0 * c5 * np.sqrt(1.5 / 2.0)
    near = float(c5[np.argmin(np.abs(prod - np.round(prod)))])
    pick.append(near)
    pick += list(synth.config_scales(1))
    pick = sorted(set(pick))
    taps["pick_scales"] = np.array(pick)
    for i, s in enumerate(pick):
        taps[f"taps_{i}"] = sample_wavelet(params, s)
    alt = MorletParams(center_frequency=0.8, bandwidth=2.0, support_radius=4.0)
    taps["alt_params"] = np.array([0.8, 2.0, 4.0])
    for i, s in enumerate([1.0, 7.7, 64.0]):
        taps[f"alt_taps_{i}"] = sample_wavelet(alt, s)
    taps["alt_scales"] = np.array([1.0, 7.7, 64.0])
    np.savez_compressed(os.path.join(OUT, "taps.npz"), **taps)

    # ---- transforms -------------------------------------------------------------------
    cases = {}

    def add(name, x32, scales, hop, wavelet, output, norm, p=None):
        p = p or params
        vals = ref_cwth(x32, scales, hop, p)
        cases[f"{name}__x"] = np.asarray(x32, dtype=np.float32)
        cases[f"{name}__scales"] = np.asarray(scales, dtype=np.float64)
        cases[f"{name}__meta"] = np.array([hop, p.center_frequency, p.bandwidth, p.support_radius])
        cases[f"{name}__kind"] = np.array([wavelet, output, norm or "none"])
        cases[f"{name}__ref"] = vals

    add("c1", synth.make_clip(1, 0), synth.config_scales(1), 16, "rmor", "abs", None)
    add("c2s", synth.make_clip(2, 0, 8000), np.geomspace(1, 128, 16), 64, "rmor", "log1p", None)
    add("c3s", synth.make_clip(3, 0, 2048), np.geomspace(1, 128, 8), 1, "rmor", "abs", None)
    x4 = synth.make_clip(4, 0, 6000)
    for h in (16, 256, 1024):
        add(f"c4s_h{h}", x4, np.geomspace(1, 256, 8), h, "rmor", "abs", None)
    add("c5s", synth.make_clip(5, 0, 6000), np.geomspace(1, 512, 12), 32, "cmor", "abs", "minmax")
    rng = np.random.default_rng(2408)
    add("ragged_1001", rng.standard_normal(1001).astype(np.float32), [1.0, 3.3, 20.0], 64,
        "cmor", "complex", None)
    add("short_5", rng.standard_normal(5).astype(np.float32), [1.0, 100.0], 2, "cmor", "complex", None)
    add("single_1", np.array([0.75], dtype=np.float32), [1.0, 2.0], 1, "cmor", "complex", None)
    add("hop_gt_n", rng.standard_normal(100).astype(np.float32), [1.5, 6.0], 128, "cmor", "complex", None)
    add("odd_hop_7", rng.standard_normal(3000).astype(np.float32), np.geomspace(1, 40, 10), 7,
        "cmor", "complex", None)
    add("alt_params", rng.standard_normal(2500).astype(np.float32), np.geomspace(2, 50, 6), 8,
        "cmor", "complex", None, MorletParams(0.8, 2.0, 4.0))
    imp = synthesize(SynthSpec("impulse", 600, 16_000.0, position=300)).samples.astype(np.float32)
    grid = make_scale_grid(500.0, 4000.0, 5, 16_000.0, params)
    add("impulse_h1", imp, grid.scales, 1, "cmor", "complex", None)
    add("impulse_h4", imp, grid.scales, 4, "cmor", "complex", None)
    add("zeros", np.zeros(777, dtype=np.float32), [2.0, 30.0], 16, "cmor", "abs", "minmax")

    # scalogram.py KATs on a reference matrix
    m = wavehop.CoefficientMatrix(cases["c5s__ref"], 32, 16_000.0, ScaleGrid(np.geomspace(1, 512, 12)))
    for mode in ("abs", "power", "log_db"):
        cases[f"mag_{mode}"] = magnitude(m, mode)
    cases["render_abs"] = render(magnitude(m, "abs")).pixels
    cases["render_abs_noflip"] = render(magnitude(m, "abs"), flip_vertical=False).pixels
    np.savez_compressed(os.path.join(OUT, "cwth.npz"), **cases)

    # ---- §8f rows: decimate / cwth_decimate / render / file formats -------------------------
    from wavehop.scalogram import write_csv, write_matrix_bin, write_pgm  # noqa: E402
    from wavehop.signal_io import decimate  # noqa: E402
    from wavehop.wavelet import cwth_decimate  # noqa: E402
    import tempfile  # noqa: E402

    fmt = {}
    rng = np.random.default_rng(2408_14302_8)
    for name, n, hop, aa in (("d_n5000_h4", 5000, 4, False), ("d_n5000_h4_aa", 5000, 4, True),
                             ("d_n4096_h16_aa", 4096, 16, True), ("d_n1001_h7_aa", 1001, 7, True),
                             ("d_n50_h64_aa", 50, 64, True), ("d_n300_h1_aa", 300, 1, True),
                             ("d_n300_h1", 300, 1, False)):
        x = rng.standard_normal(n).astype(np.float32)
        d = decimate(SignalBuffer(x.astype(np.float64), 16_000.0), hop, aa)
        fmt[f"{name}__x"] = x
        fmt[f"{name}__meta"] = np.array([hop, int(aa)], dtype=np.int64)
        fmt[f"{name}__ref"] = d.samples
        fmt[f"{name}__rate"] = np.array(d.sample_rate)
    for name, n, hop, aa, sc in (("cd_h8", 4000, 8, False, np.geomspace(1.0, 12.0, 6)),
                                 ("cd_h8_aa", 4000, 8, True, np.geomspace(1.0, 12.0, 6)),
                                 ("cd_h32_aa", 16000, 32, True, np.geomspace(1.5, 20.0, 5))):
        x = rng.standard_normal(n).astype(np.float32)
        m = cwth_decimate(SignalBuffer(x.astype(np.float64), 16_000.0), ScaleGrid(sc), params, hop, aa)
        fmt[f"{name}__x"] = x
        fmt[f"{name}__scales"] = sc
        fmt[f"{name}__meta"] = np.array([hop, int(aa), m.hop], dtype=np.int64)
        fmt[f"{name}__rate"] = np.array(m.source_rate)
        fmt[f"{name}__ref"] = m.values
    # render on float32-representable matrices, incl. exact .5 ties and a constant matrix
    v = rng.standard_normal((7, 33)).astype(np.float32)
    fmt["render_rand__v"] = v
    fmt["render_rand__flip"] = render(v.astype(np.float64)).pixels
    fmt["render_rand__noflip"] = render(v.astype(np.float64), flip_vertical=False).pixels
    ties = (np.arange(0, 511, dtype=np.float32) / 2.0).reshape(7, 73)  # scaled = k/2 exactly
    fmt["render_ties__v"] = ties
    fmt["render_ties__flip"] = render(ties.astype(np.float64)).pixels
    const = np.full((3, 5), 2.5, dtype=np.float32)
    fmt["render_const__v"] = const
    fmt["render_const__flip"] = render(const.astype(np.float64)).pixels
    # byte-exact writers
    cm = wavehop.CoefficientMatrix(cases["c5s__ref"], 32, 16_000.0, ScaleGrid(np.geomspace(1, 512, 12)))
    with tempfile.TemporaryDirectory() as td:
        write_matrix_bin(cm, os.path.join(td, "m.scg1"))
        write_pgm(render(magnitude(cm, "abs")), os.path.join(td, "m.pgm"))
        write_csv(magnitude(cm, "log_db")[:3, :10], os.path.join(td, "m.csv"))
        for ext in ("scg1", "pgm", "csv"):
            with open(os.path.join(td, f"m.{ext}"), "rb") as f:
                fmt[f"file_{ext}"] = np.frombuffer(f.read(), dtype=np.uint8)
    # wav / synth (signal_io.py:63-250) for the CLI and scan rows
    from wavehop.signal_io import read_wav, write_wav  # noqa: E402
    import struct  # noqa: E402
    for i, (kind, kw) in enumerate((("impulse", dict(position=17)), ("sine", dict(frequency=440.0, amplitude=0.3)),
                                    ("chirp", dict(f0=100.0, f1=3000.0)), ("white_noise", dict(seed=7)))):
        fmt[f"synth_{kind}"] = synthesize(SynthSpec(kind, 1000, 8000.0, **kw)).samples
    sig = SignalBuffer(np.sin(np.arange(300) * 0.05) * 0.9, 11025.0)
    with tempfile.TemporaryDirectory() as td:
        for enc in ("pcm16", "float32"):
            write_wav(sig, os.path.join(td, f"{enc}.wav"), encoding=enc)
            with open(os.path.join(td, f"{enc}.wav"), "rb") as f:
                fmt[f"wav_{enc}"] = np.frombuffer(f.read(), dtype=np.uint8)
            fmt[f"wav_{enc}__read"] = read_wav(os.path.join(td, f"{enc}.wav")).samples
        # a stereo pcm16 file with an odd-sized extra chunk (word alignment) -> mono average
        st = (np.arange(40, dtype=np.int16).reshape(20, 2) * np.array([100, -37], dtype=np.int16)).tobytes()
        fmtc = struct.pack("<HHIIHH", 1, 2, 22050, 22050 * 4, 4, 16)
        body = b"WAVE" + b"fmt " + struct.pack("<I", 16) + fmtc + b"LIST" + struct.pack("<I", 3) + b"abc\x00"
        body += b"data" + struct.pack("<I", len(st)) + st
        blob = b"RIFF" + struct.pack("<I", len(body)) + body
        with open(os.path.join(td, "st.wav"), "wb") as f:
            f.write(blob)
        fmt["wav_stereo"] = np.frombuffer(blob, dtype=np.uint8)
        fmt["wav_stereo__read"] = read_wav(os.path.join(td, "st.wav")).samples
    np.savez_compressed(os.path.join(OUT, "formats.npz"), **fmt)
    for f in ("taps.npz", "cwth.npz", "formats.npz"):
        print(f, os.path.getsize(os.path.join(OUT, f)), "bytes")


if __name__ == "__main__":
    main()
