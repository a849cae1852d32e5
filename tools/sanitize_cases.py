import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2408_14302_b200 as wh
from paper_2408_14302_b200 import synth
for cid, hop, wav, out, norm in ((2, 64, "rmor", "log1p", None), (5, 32, "cmor", "abs", "minmax"), (2, 96, "rmor", "abs", None), (3, 1, "rmor", "abs", None), (2, 1024, "rmor", "abs", None)):
    x = synth.make_batch(cid, clips=2, n=20000, start=0)
    sc = synth.config_scales(cid)
    for eng in ("umma", "simt"):
        try:
            r = wh.cwth_batch(x, sc, wh.MorletParams(), hop, wavelet=wav, output=out, norm=norm, engine=eng)
            print(cid, hop, eng, r.shape, float(np.abs(r).max()), flush=True)
        except wh.WavehopError as e:
            print(cid, hop, eng, "refused:", e, flush=True)
