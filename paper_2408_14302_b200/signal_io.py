"""Signal container, hop validation and decimation (mirrors signal_io.py:33-61, 130-156 of
the reference); decimation runs on the GPU (wh_decimate).  WAV I/O lives in ``wavio``."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import EmptySignal, InvalidHop


@dataclass(eq=False)
class SignalBuffer:
    """A discrete mono signal (signal_io.py:33-61): float64 samples + sample rate."""

    samples: np.ndarray
    sample_rate: float
    source_label: str = ""

    def __post_init__(self):
        self.samples = np.asarray(self.samples, dtype=np.float64)
        if self.samples.ndim != 1:
            raise ValueError("samples must be one-dimensional")
        if self.samples.size < 1:
            raise EmptySignal("signal has no samples")
        self.sample_rate = float(self.sample_rate)
        if not (self.sample_rate > 0 and math.isfinite(self.sample_rate)):
            raise ValueError(f"sample_rate must be positive, got {self.sample_rate}")

    def __len__(self) -> int:
        return self.samples.size

    @property
    def duration(self) -> float:
        return self.samples.size / self.sample_rate


def _check_hop(hop) -> int:
    """signal_io.py:153-156: an integer >= 1, else InvalidHop."""
    if int(hop) != hop or hop < 1:
        raise InvalidHop(f"hop must be an integer >= 1, got {hop!r}")
    return int(hop)


def decimate_device(x, hop: int, anti_alias: bool = False):
    """signal_io.py:130-150 on device clips: CUDA float32 tensor [B, N] (or [N]) ->
    [B, ceil(N/hop)] float32 (a view with 16-byte aligned rows), stream-ordered on the
    current stream.  With ``anti_alias`` the reference's FIR (firwin(10*hop+1, 0.9/hop),
    "same"-centred) is applied in float64 before the selection."""
    import ctypes

    import torch

    from . import _lib

    hop = _check_hop(hop)
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32):
        raise TypeError("decimate_device takes a CUDA float32 tensor")
    xx = x if x.dim() == 2 else x.unsqueeze(0)
    if xx.stride(-1) != 1:
        xx = xx.contiguous()
    B, n = xx.shape
    if n < 1:
        raise EmptySignal("signal has no samples")
    m = -(-n // hop)
    ld = -(-m // 4) * 4
    buf = torch.empty((B, ld), dtype=torch.float32, device=xx.device)
    stream = torch.cuda.current_stream(xx.device).cuda_stream
    ld_x = xx.stride(0) if B > 1 else n  # a size-1 batch dimension may carry stride 0
    _lib.check(_lib.load().wh_decimate(xx.device.index, ctypes.c_void_p(xx.data_ptr()), B, n,
                                       ld_x, hop, int(bool(anti_alias)),
                                       ctypes.c_void_p(buf.data_ptr()), ld, ctypes.c_void_p(stream)))
    out = buf[:, :m]
    return out if x.dim() == 2 else out[0]


def decimate(signal: SignalBuffer, hop: int, anti_alias: bool = False, *, device=None) -> SignalBuffer:
    """Drop-in for signal_io.py:130-150: keep every ``hop``-th sample from index 0 (output
    length ceil(N/hop), rate / hop); ``anti_alias`` low-passes first.  Computed on the GPU
    from the float32 samples (fp64 FIR accumulation)."""
    import torch

    hop = _check_hop(hop)
    if hop == 1 and not anti_alias:
        return SignalBuffer(signal.samples.copy(), signal.sample_rate, signal.source_label)
    dev = torch.device("cuda", 0 if device is None else int(device))
    x = torch.from_numpy(signal.samples.astype(np.float32)).to(dev)
    y = decimate_device(x, hop, anti_alias).cpu().numpy().astype(np.float64)
    return SignalBuffer(y, signal.sample_rate / hop, signal.source_label)
