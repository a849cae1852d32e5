"""Quick GPU parity check of both engines on the golden fixtures (debug helper)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_14302_b200 as wh  # noqa: E402
from paper_2408_14302_b200 import synth  # noqa: E402

g = np.load("tests/golden/cwth.npz")
names = sorted({k.split("__")[0] for k in g.files if "__" in k})
worst = {}
for engine in sys.argv[1:] or ["simt", "umma"]:
    for n in names:
        x, sc, meta, kind, ref = (g[f"{n}__{k}"] for k in ("x", "scales", "meta", "kind", "ref"))
        hop = int(meta[0])
        p = wh.MorletParams(meta[1], meta[2], meta[3])
        try:
            t0 = time.time()
            got = wh.cwth_batch(x[None], sc, p, hop, wavelet="cmor", output="complex", engine=engine)[0]
            plan = wh.get_plan(sc, p, hop, x.size, wavelet="cmor", output="complex", norm=None, clips=1,
                               device=0, engine=engine)
            rowmax = np.maximum(np.abs(ref).max(axis=1, keepdims=True), 1e-300)
            err = (np.abs(got - ref) / rowmax).max() if ref.size else 0.0
            print(f"{engine:5s} {n:12s} eng={plan.engine:5s} shape={got.shape} rowrel={err:.2e}"
                  f" {time.time()-t0:.2f}s", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"{engine:5s} {n:12s} FAILED {type(e).__name__}: {e}", flush=True)
