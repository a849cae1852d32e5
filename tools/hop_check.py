"""Both engines against the oracle over a hop list (debug helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2408_14302_b200 as wh  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2408_14302_b200 import synth  # noqa: E402

hops = [int(h) for h in (sys.argv[1].split(",") if len(sys.argv) > 1 else "3,6,12,24,48,96,192,128,256,512".split(","))]
x = synth.make_batch(2, clips=2, n=20000, start=0)
for cid, wavelet in ((2, "rmor"), (5, "cmor")):
    sc = synth.config_scales(cid)
    for hop in hops:
        ref = O.cwth_batch(x, sc, hop, wavelet=wavelet, output="abs")
        for eng in ("umma", "simt"):
            try:
                got = wh.cwth_batch(x, sc, wh.MorletParams(), hop, wavelet=wavelet, output="abs", engine=eng)
                err = (np.abs(got - ref) / np.maximum(np.abs(ref).max(-1, keepdims=True), 1e-30)).max()
                print(f"c{cid} hop {hop:4d} {eng}: {err:.2e}", flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"c{cid} hop {hop:4d} {eng}: ERR {e}", flush=True)
