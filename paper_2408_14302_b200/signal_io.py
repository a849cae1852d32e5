"""Signal container and hop validation (mirrors signal_io.py:33-61 and 153-156 of the
reference).  WAV I/O, synthesis and decimation are out of scope."""

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
