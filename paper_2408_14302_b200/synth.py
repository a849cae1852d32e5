"""Seeded synthetic clips standing in for the MIMII recordings (not in the image).

BASELINE.json names the generators; SURVEY.md §8(d) fixes their parameters.
Every clip is reproducible from (config_id, clip_index) alone via
``np.random.default_rng([config_id, clip_index])``, so any shard on any rank can
regenerate any clip and the GPU path and the oracle see the same float32 array.
"""

from __future__ import annotations

import numpy as np

SAMPLE_RATE = 16_000.0


def sinusoid_clip(config_id: int, clip: int, n: int = 16_000) -> np.ndarray:
    """c1: three sinusoids f~U(100,4000) Hz, A~U(0.1,0.5), phase~U(0,2pi) + N(0, 0.1^2)."""
    rng = np.random.default_rng([config_id, clip])
    t = np.arange(n) / SAMPLE_RATE
    f = rng.uniform(100.0, 4000.0, 3)
    a = rng.uniform(0.1, 0.5, 3)
    ph = rng.uniform(0.0, 2 * np.pi, 3)
    x = (a[:, None] * np.sin(2 * np.pi * f[:, None] * t[None, :] + ph[:, None])).sum(0)
    x += rng.normal(0.0, 0.1, n)
    return x.astype(np.float32)


def machine_noise_clip(config_id: int, clip: int, n: int = 160_000, snr_db=(-6.0, 0.0, 6.0)) -> np.ndarray:
    """c2-c5: harmonic tone (f0~U(50,500) Hz, 6 harmonics at 1/n amplitude, random phases)
    plus pink (1/f power) noise scaled to the drawn SNR.

    ``snr_db`` is a tuple to draw from, or a (lo, hi) pair given as a 2-element list
    for a uniform draw (c4)."""
    rng = np.random.default_rng([config_id, clip])
    t = np.arange(n) / SAMPLE_RATE
    f0 = rng.uniform(50.0, 500.0)
    k = np.arange(1, 7)
    ph = rng.uniform(0.0, 2 * np.pi, 6)
    tone = ((1.0 / k)[:, None] * np.sin(2 * np.pi * f0 * k[:, None] * t[None, :] + ph[:, None])).sum(0)
    white = rng.standard_normal(n)
    spec = np.fft.rfft(white)
    freqs = np.fft.rfftfreq(n, 1.0 / SAMPLE_RATE)
    spec[0] = 0.0
    spec[1:] /= np.sqrt(freqs[1:])
    pink = np.fft.irfft(spec, n)
    if isinstance(snr_db, list):
        snr = rng.uniform(snr_db[0], snr_db[1])
    else:
        snr = float(snr_db[rng.integers(len(snr_db))])
    p_tone = np.mean(tone * tone)
    p_noise = np.mean(pink * pink)
    pink *= np.sqrt(p_tone / 10.0 ** (snr / 10.0) / p_noise)
    return (tone + pink).astype(np.float32)


# BASELINE.json configs (index = config_id).  scales are geometric a0..a1.
CONFIGS = {
    1: dict(name="c1", clips=1, n=16_000, scales=(1.0, 64.0, 32), hop=16, wavelet="rmor",
            output="abs", norm=None, gen="sinusoid"),
    2: dict(name="c2", clips=64, n=160_000, scales=(1.0, 128.0, 128), hop=64, wavelet="rmor",
            output="log1p", norm=None, gen="machine", snr=(-6.0, 0.0, 6.0)),
    3: dict(name="c3", clips=8, n=160_000, scales=(1.0, 128.0, 64), hop=1, wavelet="rmor",
            output="abs", norm=None, gen="machine", snr=(-6.0, 0.0, 6.0)),
    4: dict(name="c4", clips=256, n=160_000, scales=(1.0, 256.0, 64), hop=64, wavelet="rmor",
            output="abs", norm=None, gen="machine", snr=[-6.0, 6.0], hops=(1, 16, 64, 256, 1024)),
    5: dict(name="c5", clips=4096, n=160_000, scales=(1.0, 512.0, 160), hop=32, wavelet="cmor",
            output="abs", norm="minmax", gen="machine", snr=(-6.0, 0.0, 6.0)),
}


def config_scales(cfg_id: int) -> np.ndarray:
    a0, a1, s = CONFIGS[cfg_id]["scales"]
    return np.geomspace(a0, a1, s)


def make_clip(cfg_id: int, clip: int, n: int | None = None) -> np.ndarray:
    cfg = CONFIGS[cfg_id]
    n = cfg["n"] if n is None else n
    if cfg["gen"] == "sinusoid":
        return sinusoid_clip(cfg_id, clip, n)
    return machine_noise_clip(cfg_id, clip, n, cfg["snr"])


def make_batch(cfg_id: int, clips: int | None = None, n: int | None = None, start: int = 0) -> np.ndarray:
    cfg = CONFIGS[cfg_id]
    clips = cfg["clips"] if clips is None else clips
    return np.stack([make_clip(cfg_id, start + c, n) for c in range(clips)])
