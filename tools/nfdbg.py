import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2408_14302_b200 as wh
g = np.load("tests/golden/nonfinite.npz")
for name in ("nan_h16", "inf_h64"):
    x, sc, hop, ref = g[f"{name}__x"], g[f"{name}__scales"], int(g[f"{name}__hop"]), g[f"{name}__ref"]
    for eng in ("umma", "simt"):
        try:
            got = wh.cwth_batch(x[None], sc, None, hop, wavelet="cmor", output="complex", engine=eng)[0]
        except Exception as e:
            print(name, eng, "ERR", e); continue
        for part in ("real", "imag"):
            gr, rr = getattr(got, part), getattr(ref, part)
            fin = np.isfinite(rr)
            d = np.where(fin, np.abs(gr - np.where(fin, rr, 0)), 0)
            scale = np.where(fin, np.abs(rr), 0).max(axis=1, keepdims=True)
            e = d / np.where(scale > 0, scale, 1)
            s, k = np.unravel_index(np.argmax(e), e.shape)
            print(name, eng, part, "err", e.max(), "at", s, k, "got", gr[s, k], "ref", rr[s, k], "nonfinite-got-at-finite-ref", int((~np.isfinite(gr) & fin).sum()))
