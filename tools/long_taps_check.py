"""Row error of the UMMA engine against the oracle as the taps get longer (accumulation steps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2408_14302_b200 as wh  # noqa: E402
from paper_2408_14302_b200 import synth  # noqa: E402
from oracle import oracle as O  # noqa: E402

x = synth.make_batch(5, clips=1, n=120000, start=3)
for amax in (512, 768, 1024, 1280, 1400):
    sc = np.geomspace(amax / 8, amax, 12)
    for engine in ("umma", "simt"):
        try:
            plan = wh.CwthPlan(sc, None, 32, 120000, wavelet="cmor", output="abs", max_clips=1, engine=engine)
        except Exception as e:  # noqa: BLE001
            print(amax, engine, "unsupported:", str(e)[:80])
            continue
        got = plan.execute_host(x)
        plan.close()
        ref = O.cwth_batch(x, sc, 32, wavelet="cmor", output="abs")
        den = np.abs(ref).max(axis=-1, keepdims=True)
        err = (np.abs(got - ref) / den).max(axis=-1)[0]
        print(f"a_max {amax}: {engine} worst row err {err.max():.3e} (largest scale {err[-1]:.3e})", flush=True)
