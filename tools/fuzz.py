"""Randomised parity sweep (robustness): random hops, lengths, scale grids, wavelets, outputs and
normalisations through the AUTO engine (and forced engines), each checked against the oracle.
Stops at the first failure and prints the case.  python tools/fuzz.py [n_cases] [seed]"""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2408_14302_b200 as wh  # noqa: E402
from oracle import oracle as O  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 120
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
big = len(sys.argv) > 3 and sys.argv[3] == "big"  # full-length clips (160,000+ samples), hop >= 32
hop_pool = [1, 2, 3, 4, 5, 6, 7, 8, 12, 16, 24, 31, 32, 48, 50, 64, 96, 100, 127, 128, 160, 192, 200, 255,
            256, 300, 384, 512, 640, 768, 1024, 1500]
t_start = time.time()
worst = 0.0
for i in range(n_cases):
    hop = int(rng.choice(hop_pool))
    n = int(rng.choice([1, 7, 100, 1000, 4099, 16000, 30001, 60000]))
    clips = int(rng.integers(1, 5))
    s_count = int(rng.integers(1, 48))
    a0 = float(rng.uniform(0.5, 4.0))
    a1 = float(a0 * rng.uniform(1.0, 120.0))
    if big:
        hop = int(rng.choice([h for h in hop_pool if h >= 32]))
        n = int(rng.choice([160000, 160001, 300007]))
        clips = int(rng.integers(1, 3))
        a1 = float(min(a1, 130.0))
    scales = np.unique(np.geomspace(a0, a1, s_count))
    wavelet = str(rng.choice(["cmor", "rmor"]))
    output = str(rng.choice(["complex", "abs", "power", "log1p", "log_db"]))
    norm = None
    # (min-max of log-dB values is set by the smallest |W|, whose dB value is ill-conditioned)
    if output not in ("complex", "log_db") and rng.random() < 0.3:
        norm = "minmax"
    engine = str(rng.choice(["auto", "auto", "umma", "simt"]))
    x = rng.standard_normal((clips, n)).astype(np.float32)
    case = dict(i=i, hop=hop, n=n, clips=clips, S=len(scales), a=(round(a0, 3), round(a1, 3)), wavelet=wavelet,
                output=output, norm=norm, engine=engine)
    try:
        got = wh.cwth_batch(x, scales, wh.MorletParams(), hop, wavelet=wavelet, output=output, norm=norm,
                            engine=engine)
    except wh.WavehopError as e:  # noqa: F841 -- planner refusals (forced engine) are fine
        if engine == "umma" and ("unsupported" in str(e).lower() or "UMMA engine" in str(e)):
            continue
        print("FAIL (error)", case, e, flush=True)
        sys.exit(1)
    except Exception as e:  # noqa: BLE001
        if engine == "umma" and "UMMA" in str(e):
            continue
        print("FAIL (error)", case, type(e).__name__, e, flush=True)
        sys.exit(1)
    ref = O.cwth_batch(x, scales, hop, wavelet=wavelet, output=output, norm=norm)
    assert got.shape == ref.shape == (clips, len(scales), math.ceil(n / hop)), (case, got.shape, ref.shape)
    if ref.size == 0:
        continue
    if output == "log_db" and norm is None:
        # 20 log10(|W| + 1e-12) is ill-conditioned where |W| << the row peak (zero crossings of
        # real-Morlet rows): compare the magnitudes it encodes with the row metric instead
        got, ref = 10.0 ** (got.astype(np.float64) / 20.0), 10.0 ** (ref / 20.0)
        output = "abs"
    if norm == "minmax":
        # per clip 1e-5 * max/(max - min) of the un-normalised values
        # (relative outputs) or 1e-5/(max - min) (log1p: absolute); power 2e-5, log_db in dB
        raw = O.cwth_batch(x, scales, hop, wavelet=wavelet, output=output).reshape(clips, -1)
        hi, lo = raw.max(axis=1), raw.min(axis=1)
        span = np.where(hi > lo, hi - lo, np.inf)
        base = {"log1p": 1e-5 / span, "log_db": (20.0 / np.log(10.0) * 1e-5 + 2e-5) / span,
                "power": 2e-5 * np.abs(hi) / span}.get(output, 1e-5 * np.abs(hi) / span)
        errs = np.abs(got.astype(np.float64) - ref).reshape(clips, -1).max(axis=1)
        k = int(np.argmax(errs / base))
        err, tol = float(errs[k]), float(base[k])
    elif output == "log1p":
        err = float(np.abs(got - ref).max())
        tol = 1e-5
    else:
        r2 = ref.reshape(-1, ref.shape[-1])
        g2 = got.reshape(-1, got.shape[-1])
        sc = np.abs(r2).max(axis=1)
        if r2.shape[-1] < 16:  # rows of a few frames: a cancelled sum is not a row peak
            sc = np.maximum(sc, 0.05 * np.abs(ref).reshape(clips, -1).max(axis=1).repeat(ref.shape[1]))
        ok = sc > 0
        err = float((np.abs(g2[ok] - r2[ok]).max(axis=1) / sc[ok]).max()) if ok.any() else float(np.abs(g2).max())
        tol = 2e-5 if output == "power" else 1e-5
    worst = max(worst, err / tol if tol > 0 else (0.0 if err == 0 else float("inf")))  # (constant clip: tol 0, err 0)
    if not err <= tol:
        print("FAIL (tolerance)", case, f"err {err:.3e} tol {tol:.1e}", flush=True)
        sys.exit(1)
print(f"fuzz ok: {n_cases} cases, worst err/tol {worst:.2f}, {time.time() - t_start:.0f} s", flush=True)
