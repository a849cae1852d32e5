"""paper_2408_14302_b200 -- B200-native hop-strided continuous wavelet transform (CWTH).

Drop-in for the CWTH path of the reference package ``wavehop`` 0.1.0 (arXiv 2408.14302):
``cwth_strided`` / ``cwt_fft`` / ``sample_wavelet`` keep the reference signatures; the
compute runs in hand-written sm_100a CUDA (tcgen05 split-fp16 tensor-core engine, SIMT
fp32 engine for other hops) behind the C ABI in ``include/wavehop_b200.h``.  There is no
CPU fallback.
"""

from .errors import (DeviceError, EmptySignal, InvalidCount, InvalidHop, InvalidRange,
                     InvalidScale, InvalidSpec, IoFailure, MalformedHeader, MalformedRiff,
                     TruncatedPayload, UnsupportedEncoding, WavehopError)
from .scalogram import (MAG_MODES, ScalogramImage, magnitude, read_matrix_bin, render,
                        render_device, write_csv, write_matrix_bin, write_matrix_bin_raw,
                        write_pgm)
from .signal_io import SignalBuffer, decimate, decimate_device
from .wavelet import (CoefficientMatrix, CwthPlan, MorletParams, ScaleGrid, cwt_fft, cwth_batch,
                      cwth_decimate, cwth_decimate_batch, cwth_strided, get_plan, half_width,
                      make_scale_grid, sample_wavelet, scale_to_frequency)

__version__ = "0.1.0"
