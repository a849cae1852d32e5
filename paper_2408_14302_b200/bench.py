"""Wall-clock comparison of the transform paths, GPU edition of the reference's
bench.py:1-132: same ``BenchReport`` JSON-lines schema
(bench.py:36-44), same method names, same warm-up + ``reps`` protocol and
``speedup_vs_full`` against the full transform -- every method runs through this
package's public API on the GPU (host signal in, host CoefficientMatrix out).

The DWT and the direct-summation path are not on the GPU path; asking for
them raises ValueError.
"""

from __future__ import annotations

import json
import statistics
import time
from dataclasses import asdict, dataclass

from .signal_io import SignalBuffer
from .wavelet import MorletParams, ScaleGrid, cwt_fft, cwth_decimate, cwth_strided

FULL_METHOD = "cwt_fft"


@dataclass
class BenchReport:
    method: str
    signal_length: int
    scale_count: int
    hop: int
    repetitions: int
    median_seconds: float
    min_seconds: float
    speedup_vs_full: float

    def to_json(self) -> str:
        return json.dumps(asdict(self))


def _time_repeated(fn, reps: int) -> list[float]:
    fn()  # warm-up (plan creation, filter bank build), excluded
    times = []
    for _ in range(reps):
        start = time.perf_counter()
        fn()
        times.append(time.perf_counter() - start)
    return times


def summarize(times: list[float]) -> tuple[float, float]:
    """(median, min) of a list of timings."""
    return statistics.median(times), min(times)


def bench_single(signal: SignalBuffer, grid: ScaleGrid, params: MorletParams | None = None,
                 hop: int = 128, reps: int = 5, *, include_decimate: bool = False,
                 include_dwt: bool = False, include_direct: bool = False, dwt_bank=None,
                 dwt_levels: int | None = None, threads: int = 1, device=None) -> list[BenchReport]:
    """bench.py:65-121 on the GPU: ``cwt_fft`` (the speedup reference) and ``cwth_strided``,
    optionally ``cwth_decimate``."""
    if reps < 3:
        raise ValueError(f"reps must be >= 3, got {reps}")
    if include_dwt or include_direct:
        raise ValueError("the DWT and direct-summation paths are not on the GPU path")
    params = params or MorletParams()
    jobs = [
        (FULL_METHOD, lambda: cwt_fft(signal, grid, params, threads=threads, device=device)),
        ("cwth_strided", lambda: cwth_strided(signal, grid, params, hop, threads=threads, device=device)),
    ]
    if include_decimate:
        jobs.append(("cwth_decimate",
                     lambda: cwth_decimate(signal, grid, params, hop, threads=threads, device=device)))
    measured = {name: summarize(_time_repeated(fn, reps)) for name, fn in jobs}
    full_median = measured[FULL_METHOD][0]
    return [BenchReport(method=name, signal_length=len(signal), scale_count=grid.count,
                        hop=hop if name.startswith("cwth") else 1, repetitions=reps,
                        median_seconds=measured[name][0], min_seconds=measured[name][1],
                        speedup_vs_full=full_median / measured[name][0])
            for name, _ in jobs]


def extrapolate_dataset(report: BenchReport, file_count: int) -> float:
    """bench.py:124-128: hours to process ``file_count`` files at this report's median."""
    if file_count < 1:
        raise ValueError(f"file_count must be >= 1, got {file_count}")
    return report.median_seconds * file_count / 3600.0


def reports_to_jsonl(reports: list[BenchReport]) -> str:
    return "\n".join(r.to_json() for r in reports) + "\n"
