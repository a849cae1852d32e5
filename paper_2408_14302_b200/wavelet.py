"""B200 CWTH entry points -- drop-ins for the reference's wavelet.py.

Reference (wavehop 0.1.0, /root/reference/pkg/src/wavehop):
  MorletParams      wavelet.py:32-53      ScaleGrid          wavelet.py:56-73
  CoefficientMatrix wavelet.py:76-109     make_scale_grid    wavelet.py:112-134
  sample_wavelet    wavelet.py:144-159    cwt_fft            wavelet.py:187-212
  cwth_strided      wavelet.py:215-273

Every transform here runs on the GPU through libwavehop_b200.so (include/wavehop_b200.h);
nothing falls back to the CPU.  Differences from the reference, by design:
  * arithmetic is fp32-level (split-fp16 tensor cores or fp32 SIMT) instead of float64;
    results match the reference within the tolerance stated in DESIGN.md (1e-5 of each
    row's peak); shapes, frame positions and scale order are bit-exact;
  * ``threads`` is accepted for signature compatibility and ignored (the device
    parallelises over clips, scales and frames);
  * ``cwth_batch`` adds a batched, fused-epilogue entry (log1p, per-clip min-max, real
    Morlet) for the BASELINE configurations.
"""

from __future__ import annotations

import ctypes
import math
import threading
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InvalidCount, InvalidRange, InvalidScale
from .signal_io import SignalBuffer, _check_hop


@dataclass
class MorletParams:
    """Complex Morlet parameters (wavelet.py:32-53)."""

    center_frequency: float = 1.0
    bandwidth: float = 1.5
    support_radius: float = 6.0

    def __post_init__(self):
        if not self.center_frequency > 0:
            raise ValueError("center_frequency must be positive")
        if not self.bandwidth > 0:
            raise ValueError("bandwidth must be positive")
        if not self.support_radius >= 3:
            raise ValueError("support_radius must be at least 3")


@dataclass
class ScaleGrid:
    """Strictly ascending positive scales (wavelet.py:56-73)."""

    scales: np.ndarray

    def __post_init__(self):
        self.scales = np.asarray(self.scales, dtype=np.float64)
        if self.scales.ndim != 1 or self.scales.size < 1:
            raise ValueError("scales must be a non-empty 1-D sequence")
        if not np.all(self.scales > 0):
            raise ValueError("scales must be positive")
        if not np.all(np.diff(self.scales) > 0):
            raise ValueError("scales must be strictly ascending")

    @property
    def count(self) -> int:
        return self.scales.size


@dataclass
class CoefficientMatrix:
    """Complex coefficients, rows = ascending scales, column k = translation k*hop
    (wavelet.py:76-109)."""

    values: np.ndarray
    hop: int
    source_rate: float
    scale_grid: ScaleGrid

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=np.complex128)
        if self.values.ndim != 2:
            raise ValueError("values must be a 2-D matrix")
        self.hop = _check_hop(self.hop)
        self.source_rate = float(self.source_rate)
        if not self.source_rate > 0:
            raise ValueError("source_rate must be positive")
        if self.values.shape[0] != self.scale_grid.count:
            raise ValueError(
                f"row count {self.values.shape[0]} != scale count {self.scale_grid.count}")

    @property
    def rows(self) -> int:
        return self.values.shape[0]

    @property
    def columns(self) -> int:
        return self.values.shape[1]


def make_scale_grid(f_min: float, f_max: float, count: int, sample_rate: float,
                    params: MorletParams | None = None) -> ScaleGrid:
    """wavelet.py:112-134 (host parameter arithmetic)."""
    params = params or MorletParams()
    if not (0 < f_min <= f_max < sample_rate / 2):
        raise InvalidRange(
            f"need 0 < f_min <= f_max < rate/2, got [{f_min}, {f_max}] at rate {sample_rate}")
    if count < 1:
        raise InvalidCount(f"count must be >= 1, got {count}")
    if count == 1 and f_min != f_max:
        raise InvalidCount("count == 1 needs f_min == f_max")
    freqs = np.geomspace(f_max, f_min, count)
    return ScaleGrid(params.center_frequency * sample_rate / freqs)


def scale_to_frequency(scale: float, params: MorletParams, sample_rate: float) -> float:
    """wavelet.py:137-141."""
    if not (scale > 0 and math.isfinite(scale)):
        raise InvalidScale(f"scale must be positive and finite, got {scale!r}")
    return params.center_frequency * sample_rate / scale


def half_width(scale: float, params: MorletParams | None = None) -> int:
    """wavelet.py:154 (L = ceil(R * a * sqrt(B / 2)) in float64), via the C ABI."""
    params = params or MorletParams()
    out = ctypes.c_int64()
    _lib.check(_lib.load().wh_half_width(float(scale), params.bandwidth, params.support_radius,
                                         ctypes.byref(out)))
    return out.value


# --------------------------------------------------------------------------------------
# Plans
# --------------------------------------------------------------------------------------

def _device_index(device) -> int:
    if device is None:
        return 0
    if isinstance(device, int):
        return device
    idx = getattr(device, "index", None)
    if idx is not None:
        return idx
    s = str(device)
    return int(s.split(":")[1]) if ":" in s else 0


class CwthPlan:
    """A device plan: filter bank on the GPU + engine choice for fixed
    (scales, params, hop, n_samples, wavelet, output, norm).  Wraps wh_plan_*."""

    def __init__(self, scales, params: MorletParams | None = None, hop: int = 128,
                 n_samples: int = 1, *, wavelet: str = "cmor", output: str = "complex",
                 norm=None, max_clips: int = 1, device=None, engine: str = "auto"):
        params = params or MorletParams()
        hop = _check_hop(hop)
        self.scales = np.ascontiguousarray(np.asarray(scales, dtype=np.float64))
        self.params, self.hop, self.n_samples = params, hop, int(n_samples)
        self.wavelet, self.output, self.norm = wavelet, output, norm
        self.max_clips, self.device = int(max_clips), _device_index(device)
        lib = _lib.load()
        handle = ctypes.c_void_p()
        if wavelet not in _lib.WAVELETS:
            raise ValueError(f"wavelet must be one of {tuple(_lib.WAVELETS)}")
        if output not in _lib.OUTPUTS:
            raise ValueError(f"output must be one of {tuple(_lib.OUTPUTS)}")
        if norm not in _lib.NORMS:
            raise ValueError("norm must be None, 'minmax', 'render' or 'render_noflip'")
        _lib.check(lib.wh_plan_create(
            ctypes.byref(handle), self.device,
            self.scales.ctypes.data_as(ctypes.c_void_p), int(self.scales.size),
            params.center_frequency, params.bandwidth, params.support_radius,
            _lib.WAVELETS[wavelet], hop, self.n_samples, self.max_clips,
            _lib.OUTPUTS[output], _lib.NORMS[norm], _lib.ENGINES[engine]))
        self._h = handle
        self._lock = threading.Lock()
        f = ctypes.c_int64()
        _lib.check(lib.wh_plan_frames(self._h, ctypes.byref(f)))
        self.frames = f.value
        e = ctypes.c_int32()
        _lib.check(lib.wh_plan_engine(self._h, ctypes.byref(e)))
        self.engine = _lib.ENGINE_NAMES[e.value]

    # -- queries --------------------------------------------------------------------
    @property
    def out_shape_per_clip(self):
        return (self.scales.size, self.frames)

    @property
    def out_dtype(self):
        """numpy dtype of the output: complex64, float32, or uint8 for render plans."""
        if self.norm in ("render", "render_noflip"):
            return np.dtype(np.uint8)
        return np.dtype(np.complex64 if self.output == "complex" else np.float32)

    def launches(self, clips: int) -> int:
        n = ctypes.c_int64()
        _lib.check(_lib.load().wh_plan_launches(self._h, int(clips), ctypes.byref(n)))
        return n.value

    def mma_flops(self, clips: int) -> float:
        """Tensor-core flops one execute() of ``clips`` clips issues (0 for the SIMT engine)."""
        f = ctypes.c_double()
        _lib.check(_lib.load().wh_plan_mma_flops(self._h, int(clips), ctypes.byref(f)))
        return f.value

    def taps(self, index: int) -> np.ndarray:
        """Device-built taps of scale ``index`` as complex64 (2L+1 values)."""
        L = half_width(self.scales[index], self.params)
        re = np.empty(2 * L + 1, dtype=np.float32)
        im = np.empty(2 * L + 1, dtype=np.float32)
        h = ctypes.c_int64()
        _lib.check(_lib.load().wh_plan_taps(self._h, int(index), re.ctypes.data_as(ctypes.c_void_p),
                                            im.ctypes.data_as(ctypes.c_void_p), re.size,
                                            ctypes.byref(h)))
        return re + 1j * im.astype(np.complex64)

    def profile(self, enable: bool = True):
        """Diagnostics: enable the UMMA kernel's per-role wait counters and return (and
        reset) the counters accumulated so far as {role: {wait slots, total}} cycles."""
        buf = (ctypes.c_uint64 * 20)()
        _lib.check(_lib.load().wh_plan_profile(self._h, int(enable), buf, 20))
        roles = ("producer", "mma", "converter", "epilogue", "relay")
        return {r: list(buf[i * 4:(i + 1) * 4]) for i, r in enumerate(roles)}

    def trace(self, enable: bool = True, per_cta: bool = False):
        """Diagnostics: CTA-0 timeline of the UMMA kernel, int64 [16 events, 32 units] of
        clock64; with ``per_cta`` also int64 [256, 2] %globaltimer ns at CTA entry / exit."""
        n = 16 * 32 + 2 * 256
        buf = (ctypes.c_int64 * n)()
        _lib.check(_lib.load().wh_plan_trace(self._h, int(enable), buf, n))
        a = np.array(buf, dtype=np.int64)
        t = a[:512].reshape(16, 32)
        return (t, a[512:].reshape(256, 2)) if per_cta else t

    # -- execution ------------------------------------------------------------------
    def _check_input(self, clips: int, n: int):
        if n != self.n_samples:
            raise ValueError(f"plan built for {self.n_samples} samples, got {n}")
        if clips > self.max_clips:
            raise ValueError(f"plan built for at most {self.max_clips} clips, got {clips}")

    def execute_host(self, x: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """Host float32 [B, N] -> host output; H2D, kernels and D2H inside (wh_execute_host)."""
        x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float32)
        B, n = x.shape
        self._check_input(B, n)
        shape = (B, self.scales.size, self.frames)
        dtype = self.out_dtype
        if out is None:
            out = np.empty(shape, dtype=dtype)
        elif out.shape != shape or out.dtype != dtype or not out.flags.c_contiguous:
            raise ValueError("out has the wrong shape/dtype/layout")
        with self._lock:
            _lib.check(_lib.load().wh_execute_host(self._h, x.ctypes.data_as(ctypes.c_void_p), B,
                                                   out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def execute(self, x, out=None, stream=None):
        """Device torch tensor float32 [B, N] (CUDA) -> device output tensor, stream-ordered
        on ``stream`` (default: torch's current stream); no host synchronisation."""
        import torch

        if not (isinstance(x, torch.Tensor) and x.is_cuda):
            raise TypeError("execute() takes a CUDA tensor; use execute_host() for host arrays")
        if x.dtype != torch.float32:
            raise TypeError("x must be float32")
        if x.dim() == 1:
            x = x.unsqueeze(0)
        if x.stride(-1) != 1:
            x = x.contiguous()
        B, n = x.shape
        self._check_input(B, n)
        shape = (B, self.scales.size, self.frames)
        dtype = {np.dtype(np.uint8): torch.uint8, np.dtype(np.complex64): torch.complex64,
                 np.dtype(np.float32): torch.float32}[self.out_dtype]
        if out is None:
            out = torch.empty(shape, dtype=dtype, device=x.device)
        elif tuple(out.shape) != shape or out.dtype != dtype or not out.is_contiguous():
            raise ValueError("out has the wrong shape/dtype/layout")
        if stream is None:
            stream = torch.cuda.current_stream(x.device)
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        ld_x = x.stride(0) if B > 1 else n  # a size-1 batch dimension may carry stride 0
        with self._lock:
            if not self._h:
                raise ValueError("plan is closed")
            _lib.check(_lib.load().wh_execute(self._h, ctypes.c_void_p(x.data_ptr()), B, ld_x,
                                              ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(handle)))
        return out

    def close(self):
        """Release the plan's device memory (waits for a call in flight on another thread).
        A plan's min-max / render workspace serves one launch at a time: calls on one plan are
        serialised by its lock, and wh_execute's launches on different streams must not
        overlap (wh_execute_host orders its own two streams)."""
        lock = getattr(self, "_lock", None)
        if lock is None:
            return
        with lock:
            if getattr(self, "_h", None):
                _lib.load().wh_plan_destroy(self._h)
                self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_plans: "OrderedDict[tuple, CwthPlan]" = OrderedDict()
_plans_lock = threading.Lock()
_PLAN_CACHE = 16


def get_plan(scales, params, hop, n_samples, *, wavelet, output, norm, clips, device, engine):
    params = params or MorletParams()
    key = (tuple(np.asarray(scales, dtype=np.float64).tolist()), params.center_frequency,
           params.bandwidth, params.support_radius, int(hop), int(n_samples), wavelet, output,
           norm, _device_index(device), engine)
    with _plans_lock:
        plan = _plans.get(key)
        if plan is not None and plan.max_clips >= clips:
            _plans.move_to_end(key)
            return plan
        # a replaced or evicted plan is not closed here: another thread may still hold it (it
        # got it from this cache); its device memory is released when the last reference goes
        # (CwthPlan.__del__ -> close, which waits for a running call through the plan's lock)
        plan = CwthPlan(scales, params, hop, n_samples, wavelet=wavelet, output=output, norm=norm,
                        max_clips=max(clips, 1), device=device, engine=engine)
        _plans[key] = plan
        while len(_plans) > _PLAN_CACHE:
            _plans.popitem(last=False)
        return plan


# --------------------------------------------------------------------------------------
# Entry points
# --------------------------------------------------------------------------------------

def cwth_batch(x, scales, params: MorletParams | None = None, hop: int = 128, *,
               wavelet: str = "cmor", output: str = "complex", norm=None, device=None,
               engine: str = "auto", out=None):
    """Batched CWTH with a fused epilogue.

    x: float32 [B, N] (or [N]) as a numpy array (host; returns numpy) or a CUDA torch
    tensor (returns a CUDA tensor, stream-ordered on the current stream).  Output shape
    (B, S, ceil(N/hop)); complex64 for output="complex", else float32."""
    hop = _check_hop(hop)
    try:
        import torch
        is_tensor = isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        is_tensor = False
    if is_tensor:
        if not x.is_cuda:
            raise TypeError("torch tensors must live on a CUDA device")
        xx = x if x.dim() == 2 else x.unsqueeze(0)
        plan = get_plan(scales, params, hop, xx.shape[1], wavelet=wavelet, output=output,
                        norm=norm, clips=xx.shape[0], device=x.device, engine=engine)
        res = plan.execute(xx, out=out)
        return res if x.dim() == 2 else res[0]
    arr = np.asarray(x, dtype=np.float32)
    xx = np.atleast_2d(arr)
    plan = get_plan(scales, params, hop, xx.shape[1], wavelet=wavelet, output=output, norm=norm,
                    clips=xx.shape[0], device=device, engine=engine)
    res = plan.execute_host(xx, out=out)
    return res if arr.ndim == 2 else res[0]


def sample_wavelet(params: MorletParams, scale: float, *, device=None) -> np.ndarray:
    """wavelet.py:144-159: the conjugated, 1/sqrt(a)-normalised taps -- built on the
    device (fp64 math, fp32 storage) and read back as complex128."""
    if not (scale > 0 and math.isfinite(scale)):
        raise InvalidScale(f"scale must be positive and finite, got {scale!r}")
    plan = get_plan([float(scale)], params, 1, 1, wavelet="cmor", output="complex", norm=None,
                    clips=1, device=device, engine="simt")
    return plan.taps(0).astype(np.complex128)


def cwth_strided(signal: SignalBuffer, grid: ScaleGrid, params: MorletParams | None = None,
                 hop: int = 128, *, threads: int = 1, device=None,
                 engine: str = "auto") -> CoefficientMatrix:
    """Drop-in for wavelet.py:215-273: coefficients only at translations 0, hop, 2*hop, ...

    Column k equals column k*hop of the full transform.  Computed on the GPU in
    fp32-level arithmetic; returned as complex128 like the reference."""
    params = params or MorletParams()
    hop = _check_hop(hop)
    vals = cwth_batch(signal.samples.astype(np.float32)[None, :], grid.scales, params, hop,
                      wavelet="cmor", output="complex", device=device, engine=engine)[0]
    return CoefficientMatrix(vals.astype(np.complex128), hop, signal.sample_rate,
                             ScaleGrid(grid.scales.copy()))


def cwth_decimate(signal: SignalBuffer, grid: ScaleGrid, params: MorletParams | None = None,
                  hop: int = 128, anti_alias: bool = False, *, threads: int = 1, device=None,
                  engine: str = "auto") -> CoefficientMatrix:
    """Drop-in for wavelet.py:276-294: decimate by ``hop`` (signal_io.py:130-150, optional
    anti-alias FIR) on the device, then the full hop = 1 transform of the decimated signal
    -- the scales act on the decimated rate.  Returns the reference's matrix: hop = ``hop``,
    source_rate = rate / hop."""
    params = params or MorletParams()
    hop = _check_hop(hop)
    vals = cwth_decimate_batch(signal.samples.astype(np.float32)[None, :], grid.scales, params,
                               hop, anti_alias, wavelet="cmor", output="complex", device=device,
                               engine=engine)[0]
    return CoefficientMatrix(vals.astype(np.complex128), hop, signal.sample_rate / hop,
                             ScaleGrid(grid.scales.copy()))


def cwth_decimate_batch(x, scales, params: MorletParams | None = None, hop: int = 128,
                        anti_alias: bool = False, *, wavelet: str = "cmor",
                        output: str = "complex", norm=None, device=None, engine: str = "auto"):
    """Batched cwth_decimate: host float32 [B, N] -> (B, S, ceil(N/hop)) on the device
    (wh_decimate, then a hop-1 plan on the decimated clips; nothing leaves the GPU between
    the two)."""
    import torch

    from .signal_io import decimate_device

    hop = _check_hop(hop)
    arr = np.asarray(x, dtype=np.float32)
    xx = np.atleast_2d(arr)
    dev = torch.device("cuda", _device_index(device))
    xd = torch.from_numpy(np.ascontiguousarray(xx)).to(dev)
    dec = decimate_device(xd, hop, anti_alias)
    plan = get_plan(scales, params, 1, dec.shape[1], wavelet=wavelet, output=output, norm=norm,
                    clips=dec.shape[0], device=dev.index, engine=engine)
    res = plan.execute(dec).cpu().numpy()
    return res if arr.ndim == 2 else res[0]


def cwt_fft(signal: SignalBuffer, grid: ScaleGrid, params: MorletParams | None = None, *,
            threads: int = 1, device=None, engine: str = "auto") -> CoefficientMatrix:
    """Drop-in for wavelet.py:187-212 (the full hop = 1 transform).  The reference uses an
    FFT per row; on the B200 the direct tensor-core correlation at hop = 1 is used
    (same coefficients within tolerance)."""
    params = params or MorletParams()
    vals = cwth_batch(signal.samples.astype(np.float32)[None, :], grid.scales, params, 1,
                      wavelet="cmor", output="complex", device=device, engine=engine)[0]
    return CoefficientMatrix(vals.astype(np.complex128), 1, signal.sample_rate,
                             ScaleGrid(grid.scales.copy()))
