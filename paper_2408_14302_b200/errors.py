"""Exception hierarchy mirroring the reference's errors.py (wavehop 0.1.0, errors.py:4-67).

Only the types the CWTH path raises are needed for the drop-in; the names and bases
match the reference so ``except InvalidHop`` / ``except ValueError`` behave the same.
"""


class WavehopError(Exception):
    """Base class for every error this package raises on purpose (errors.py:4)."""


class EmptySignal(WavehopError):
    """A signal must contain at least one sample (errors.py:18)."""


class InvalidHop(WavehopError, ValueError):
    """Hop size must be an integer >= 1 (errors.py:24)."""


class InvalidScale(WavehopError, ValueError):
    """Wavelet scale must be a positive finite number (errors.py:40)."""


class DeviceError(WavehopError, RuntimeError):
    """The CUDA library failed or no B200 device is available (no reference analogue:
    the reference has no device; this path never falls back to the CPU)."""


class InvalidRange(WavehopError, ValueError):
    """Frequency range for a scale grid is out of order or out of band (errors.py:32)."""


class InvalidCount(WavehopError, ValueError):
    """Scale count is not usable for the requested range (errors.py:36)."""


class MalformedRiff(WavehopError):
    """WAV container is structurally broken (errors.py:10)."""


class UnsupportedEncoding(WavehopError):
    """WAV encoding other than 16-bit PCM or 32-bit IEEE float (errors.py:14)."""


class InvalidSpec(WavehopError, ValueError):
    """Synthesis spec violates its constraints (errors.py:28)."""


class MalformedHeader(WavehopError):
    """Coefficient-matrix file header is invalid (errors.py:58)."""


class TruncatedPayload(WavehopError):
    """Coefficient-matrix file ends before the declared payload (errors.py:62)."""


class IoFailure(WavehopError):
    """Reading or writing a file failed (errors.py:66)."""
