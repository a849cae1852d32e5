"""CPU oracle for the CWTH hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module; the product package
(``paper_2408_14302_b200``) never does.  It restates the reference package
``wavehop`` 0.1.0 (/root/reference/pkg/src/wavehop, read-only, not available on
the GPU box) in float64:

* ``wh_oracle.c`` (built into ``libwh_oracle.so`` by ``oracle/Makefile``) holds the
  per-row kernels and a pthread batch driver;
* this module adds the row router of ``wavelet.py:240-260`` (direct vs FFT row,
  ``_kernels.py:121``) for timing the reference's own CPU cost, and a numpy
  restatement of the polyphase backend (``_kernels.py:28-62``).

Pinned against the reference: ``tests/test_oracle_golden.py`` compares every
entry point with ``tests/golden/*.npz``, generated from the unmodified reference
by ``oracle/gen_golden.py``.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libwh_oracle.so")
_lib = None

WAVELETS = {"cmor": 0, "rmor": 1}
OUTPUTS = {"complex": 0, "abs": 1, "power": 2, "log_db": 3, "log1p": 4}
NORMS = {None: 0, "none": 0, "minmax": 1}
DIRECT_TO_FFT_COST_RATIO = 8.0  # _kernels.py:121


def build() -> str:
    """Compile libwh_oracle.so in place (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        d, i64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_int
        p = ctypes.c_void_p
        L.who_half_width.restype = i64
        L.who_half_width.argtypes = [d, d, d]
        L.who_sample_wavelet.restype = None
        L.who_sample_wavelet.argtypes = [d, d, d, d, p, p]
        L.who_strided_correlate.restype = None
        L.who_strided_correlate.argtypes = [p, p, p, i64, i64, i64, p, p]
        L.who_strided_correlate_symmetric.restype = None
        L.who_strided_correlate_symmetric.argtypes = [p, p, p, i64, i64, i64, p, p]
        L.who_cwth_batch.restype = i32
        L.who_cwth_batch.argtypes = [p, i64, i64, p, i64, d, d, d, i64, i32, i32, i32, p, i32]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def half_width(scale: float, bandwidth: float = 1.5, support_radius: float = 6.0) -> int:
    """wavelet.py:154."""
    return int(lib().who_half_width(scale, bandwidth, support_radius))


def sample_wavelet(scale: float, center_frequency: float = 1.0, bandwidth: float = 1.5,
                   support_radius: float = 6.0) -> np.ndarray:
    """wavelet.py:144-159; complex128 taps of length 2L+1."""
    L = half_width(scale, bandwidth, support_radius)
    re = np.empty(2 * L + 1)
    im = np.empty(2 * L + 1)
    lib().who_sample_wavelet(scale, center_frequency, bandwidth, support_radius, _ptr(re), _ptr(im))
    return re + 1j * im


def strided_correlate(xpad, taps_re, taps_im, hop, frames):
    """_kernels.py:76-91 (generic kernel)."""
    xpad = np.ascontiguousarray(xpad, dtype=np.float64)
    taps_re = np.ascontiguousarray(taps_re, dtype=np.float64)
    taps_im = np.ascontiguousarray(taps_im, dtype=np.float64)
    assert xpad.size >= (frames - 1) * hop + taps_re.size
    ore, oim = np.empty(frames), np.empty(frames)
    lib().who_strided_correlate(_ptr(xpad), _ptr(taps_re), _ptr(taps_im), taps_re.size, hop,
                                frames, _ptr(ore), _ptr(oim))
    return ore, oim


def strided_correlate_symmetric(xpad, re_half, im_half, hop, frames):
    """_kernels.py:93-112 (folded kernel)."""
    xpad = np.ascontiguousarray(xpad, dtype=np.float64)
    re_half = np.ascontiguousarray(re_half, dtype=np.float64)
    im_half = np.ascontiguousarray(im_half, dtype=np.float64)
    half = re_half.size - 1
    assert xpad.size >= (frames - 1) * hop + 2 * half + 1
    ore, oim = np.empty(frames), np.empty(frames)
    lib().who_strided_correlate_symmetric(_ptr(xpad), _ptr(re_half), _ptr(im_half), half, hop,
                                          frames, _ptr(ore), _ptr(oim))
    return ore, oim


def strided_correlate_numpy(xpad, taps_re, taps_im, hop, frames):
    """Numpy restatement of the polyphase backend, _kernels.py:28-62."""
    width = taps_re.shape[0]
    if hop <= 2:
        stride = xpad.strides[0]
        windows = np.lib.stride_tricks.as_strided(
            xpad, shape=(frames, width), strides=(stride * hop, stride), writeable=False)
        return windows @ taps_re, windows @ taps_im
    blocks = -(-width // hop)
    needed = (frames + blocks - 1) * hop
    if xpad.size < needed:
        xpad = np.concatenate([xpad, np.zeros(needed - xpad.size)])
    x2d = xpad[:needed].reshape(frames + blocks - 1, hop)
    taps2d = np.zeros((2, blocks * hop))
    taps2d[0, :width] = taps_re
    taps2d[1, :width] = taps_im
    products = np.tensordot(x2d, taps2d.reshape(2, blocks, hop), axes=([1], [2]))
    out_re = np.zeros(frames)
    out_im = np.zeros(frames)
    for q in range(blocks):
        out_re += products[q: q + frames, 0, q]
        out_im += products[q: q + frames, 1, q]
    return out_re, out_im


def cwth_batch(x, scales, hop, *, wavelet="cmor", output="complex", norm=None,
               center_frequency=1.0, bandwidth=1.5, support_radius=6.0, threads=None):
    """Direct-route CWTH of every clip + epilogue, float64.

    x: float32 [B, N] (or [N]).  Returns float64 [B, S, F] (real outputs) or
    complex128 [B, S, F] (output="complex").  Restates wavelet.py:215-273 with
    every row on the folded direct kernel (_kernels.py:93-112), then
    scalogram.py:51-64 / the BASELINE extensions."""
    x = np.asarray(x, dtype=np.float32)
    squeeze = x.ndim == 1
    x = np.ascontiguousarray(np.atleast_2d(x))
    B, N = x.shape
    scales = np.ascontiguousarray(scales, dtype=np.float64)
    S = scales.size
    F = -(-N // hop) if hop >= 1 else 0
    if threads is None:
        threads = max(1, len(os.sched_getaffinity(0)))
    cplx = output == "complex"
    out = np.empty((B, S, F, 2) if cplx else (B, S, F), dtype=np.float64)
    rc = lib().who_cwth_batch(_ptr(x), B, N, _ptr(scales), S, center_frequency, bandwidth,
                              support_radius, hop, WAVELETS[wavelet], OUTPUTS[output], NORMS[norm],
                              _ptr(out), threads)
    if rc == 1:
        raise ValueError(f"hop must be an integer >= 1, got {hop!r}")
    if rc == 2:
        raise ValueError("scale must be positive and finite")
    if rc != 0:
        raise ValueError("invalid arguments")
    if cplx:
        out = out[..., 0] + 1j * out[..., 1]
    return out[0] if squeeze else out


# --- routed restatement (reference cost model), used for CPU-baseline timing ----------

def cwth_strided_routed(x, scales, hop, center_frequency=1.0, bandwidth=1.5,
                        support_radius=6.0, backend="numba"):
    """Per-clip restatement of wavelet.py:215-273 including its row router.

    Rows whose direct cost exceeds 8*M*log2(M) go to the FFT route
    (wavelet.py:249,257-260,313-323); the rest to the folded C kernel
    (backend="numba", _kernels.py:93-112) or the numpy polyphase backend
    (backend="numpy", _kernels.py:28-62).  Returns complex128 (S, F)."""
    import scipy.fft as sfft

    x = np.asarray(x, dtype=np.float64)
    n = x.size
    frames = -(-n // hop)
    taps_per_row = [sample_wavelet(s, center_frequency, bandwidth, support_radius) for s in scales]
    longest = max(t.size for t in taps_per_row)
    fft_len = sfft.next_fast_len(n + longest - 1)
    fft_unit = DIRECT_TO_FFT_COST_RATIO * fft_len * math.log2(fft_len)
    max_half = longest // 2
    xpad = np.zeros(max_half + n + max_half + 2 * hop)
    xpad[max_half:max_half + n] = x
    spectrum = None
    if any(frames * t.size > fft_unit for t in taps_per_row):
        spectrum = sfft.fft(x, fft_len)
    out = np.empty((len(scales), frames), dtype=np.complex128)
    for row, taps in enumerate(taps_per_row):
        half = taps.size // 2
        if frames * taps.size > fft_unit:
            kernel = sfft.fft(taps[::-1], fft_len)
            dense = sfft.ifft(spectrum * kernel)[half:half + n]
            out[row] = dense[::hop]
            continue
        base = xpad[max_half - half:]
        if backend == "numba":
            re, im = strided_correlate_symmetric(base, taps.real[half:], taps.imag[half:], hop, frames)
        else:
            re, im = strided_correlate_numpy(base, np.ascontiguousarray(taps.real),
                                             np.ascontiguousarray(taps.imag), hop, frames)
        out[row] = re + 1j * im
    return out


def epilogue(values: np.ndarray, wavelet: str, output: str, norm=None) -> np.ndarray:
    """scalogram.py:51-64 magnitude + BASELINE extensions, on one clip's (S, F) complex."""
    if output == "complex":
        return values.real + 0j if wavelet == "rmor" else values
    mag = np.abs(values.real) if wavelet == "rmor" else np.abs(values)
    if output == "abs":
        res = mag
    elif output == "power":
        res = mag * mag
    elif output == "log_db":
        res = 20.0 * np.log10(mag + 1e-12)
    else:
        res = np.log1p(mag)
    if norm == "minmax":
        lo, hi = res.min(), res.max()
        res = np.zeros_like(res) if hi == lo else (res - lo) * (1.0 / (hi - lo))
    return res


# ---- decimation, render, SCG1 (restated, float64) -------------------

def firwin_lowpass(numtaps: int, cutoff: float) -> np.ndarray:
    """scipy.signal.firwin(numtaps, cutoff) with its defaults, as the reference calls it
    (signal_io.py:144; scipy is an unpinned third-party dependency, pkg/pyproject.toml:10-14):
    the published window method -- ideal low-pass cutoff*sinc(cutoff*(n - (T-1)/2)) times the
    symmetric Hamming window 0.54 - 0.46*cos(2*pi*n/(T-1)), scaled to unit gain at DC."""
    n = np.arange(numtaps, dtype=np.float64)
    m = n - 0.5 * (numtaps - 1)
    h = cutoff * np.sinc(cutoff * m)
    if numtaps > 1:
        h = h * (0.54 - 0.46 * np.cos(2.0 * np.pi * n / (numtaps - 1)))
    return h / h.sum()


def decimate(x: np.ndarray, hop: int, anti_alias: bool = False) -> np.ndarray:
    """signal_io.py:130-150: [B, N] (or [N]) float64 -> every hop-th sample from index 0;
    with ``anti_alias`` the FIR firwin(10*hop+1, 0.9/hop) is applied first as a "same"-
    centred linear convolution (fftconvolve mode="same" keeps full[(T-1)//2 : ... + N])."""
    x = np.asarray(x, dtype=np.float64)
    single = x.ndim == 1
    xx = np.atleast_2d(x)
    if anti_alias:
        h = firwin_lowpass(10 * hop + 1, 0.9 / hop)
        c = (h.size - 1) // 2
        xx = np.stack([np.convolve(row, h, mode="full")[c:c + row.size] for row in xx])
    out = xx[:, ::hop].copy()
    return out[0] if single else out


def cwth_decimate_batch(x, scales, hop, anti_alias=False, *, wavelet="cmor", output="complex",
                        norm=None, center_frequency=1.0, bandwidth=1.5, support_radius=6.0):
    """wavelet.py:276-294: decimate (above), then the full hop = 1 transform of the
    decimated signal (direct f64 oracle; the reference's FFT route agrees to ~1e-12)."""
    d = decimate(np.atleast_2d(np.asarray(x, dtype=np.float64)), hop, anti_alias)
    if not anti_alias:  # selection keeps float32 samples exact: the C batch oracle applies
        return cwth_batch(d.astype(np.float32), scales, 1, wavelet=wavelet, output=output,
                          norm=norm, center_frequency=center_frequency, bandwidth=bandwidth,
                          support_radius=support_radius)
    # the filtered signal is not float32-representable: float64 per-clip route
    vals = np.stack([cwth_strided_routed(row, scales, 1, center_frequency, bandwidth, support_radius)
                     for row in d])
    return np.stack([epilogue(v, wavelet, output, norm) for v in vals])


def render(values: np.ndarray, flip_vertical: bool = True) -> np.ndarray:
    """scalogram.py:67-86 -> uint8 pixels: (v - lo) * (255 / (hi - lo)), floor(+0.5), clip;
    constant -> zeros; flip reverses the rows."""
    values = np.asarray(values, dtype=np.float64)
    lo, hi = values.min(), values.max()
    if hi == lo:
        px = np.zeros(values.shape, dtype=np.uint8)
    else:
        px = np.clip(np.floor((values - lo) * (255.0 / (hi - lo)) + 0.5), 0, 255).astype(np.uint8)
    return px[::-1] if flip_vertical else px


def scg1_bytes(values: np.ndarray, hop: int, source_rate: float, scales: np.ndarray) -> bytes:
    """scalogram.py:100-106: "SCG1" | <III d (rows, cols, hop, rate) | f64 scales | c8 payload."""
    import struct

    values = np.asarray(values)
    rows, cols = values.shape
    return (b"SCG1" + struct.pack("<III d", rows, cols, hop, source_rate)
            + np.asarray(scales, dtype="<f8").tobytes() + values.astype("<c8").tobytes())
