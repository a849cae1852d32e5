"""Generate tests/golden/nonfinite.npz from the UNMODIFIED reference: cwth_strided
(wavelet.py:215-273) on signals holding NaN / +inf / -inf samples.

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden_nonfinite.py

The reference propagates a non-finite sample to exactly the coefficients whose support
[k*hop - L_s, k*hop + L_s] contains it (its direct kernels, _kernels.py:76-112, sum x * tap
over that support); the cases are chosen so that no row takes the FFT route (checked
below), which would spread it over the whole row.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from wavehop import MorletParams, ScaleGrid, SignalBuffer, cwth_strided  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")

CASES = {
    # name: (n, hop, scales, {position: value}, seed)
    "nan_h16": (4000, 16, np.geomspace(1, 64, 8), {1000: np.nan}, 1),
    "inf_h16": (4000, 16, np.geomspace(1, 64, 8), {1000: np.inf, 2500: -np.inf}, 2),
    "mixed_h16": (4000, 16, np.geomspace(1, 64, 8), {700: np.nan, 701: np.inf, 3000: -np.inf}, 3),
    "inf_h64": (8000, 64, np.geomspace(1, 128, 16), {5000: np.inf, 5003: np.inf}, 4),
    "nan_inf_h32": (12000, 32, np.geomspace(1, 256, 12), {100: np.inf, 6000: np.nan, 11999: -np.inf}, 5),
    "edge_h64": (8000, 64, np.geomspace(1, 128, 16), {0: -np.inf, 7999: np.nan}, 6),
}


def main():
    out = {}
    params = MorletParams()
    for name, (n, hop, scales, bad, seed) in CASES.items():
        x = np.random.default_rng(seed).uniform(-1.0, 1.0, n).astype(np.float32)
        for pos, v in bad.items():
            x[pos] = v
        with np.errstate(invalid="ignore", over="ignore"):
            ref = cwth_strided(SignalBuffer(x.astype(np.float64), 16_000.0), ScaleGrid(scales), params, hop).values
        # coherence: the non-finite set is exactly the support rule (no FFT-routed row)
        F = ref.shape[1]
        for s, a in enumerate(scales):
            L = math.ceil(6.0 * a * math.sqrt(1.5 / 2.0))
            exp = np.zeros(F, bool)
            for pos in bad:
                k = np.arange(F)
                exp |= np.abs(k * hop - pos) <= L
            got = ~np.isfinite(ref[s])
            assert np.array_equal(got, exp), (name, s)
        out[f"{name}__x"] = x
        out[f"{name}__scales"] = scales
        out[f"{name}__hop"] = np.array(hop)
        out[f"{name}__ref"] = ref
    np.savez_compressed(os.path.join(OUT, "nonfinite.npz"), **out)
    print("wrote", os.path.join(OUT, "nonfinite.npz"), len(CASES), "cases")


if __name__ == "__main__":
    main()
