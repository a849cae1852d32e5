"""One fuzz case by hand (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2408_14302_b200 as wh  # noqa: E402
from oracle import oracle as O  # noqa: E402

hop, n, S = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(5)
x = rng.standard_normal((1, n)).astype(np.float32)
sc = np.geomspace(0.876, 51.487, S)
for wavelet, output in (("cmor", "power"), ("rmor", "abs")):
    plan = wh.CwthPlan(sc, None, hop, n, wavelet=wavelet, output=output, max_clips=1, engine="umma")
    got = plan.execute_host(x)
    plan.close()
    ref = O.cwth_batch(x, sc, hop, wavelet=wavelet, output=output)
    den = np.abs(ref).max(axis=-1, keepdims=True)
    print(hop, n, wavelet, output, "err", float((np.abs(got - ref) / np.where(den > 0, den, 1)).max()), "got[0,:2]", got[0, -1, :], "ref", ref[0, -1, :], flush=True)
