"""Driver for ncu captures of the small kernels: c2-shaped decimate (selection and the
anti-alias FIR), the fused render map, and the SIMT engine (hop 100: lcm(100, 64) > 192)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_14302_b200 as wh  # noqa: E402
from paper_2408_14302_b200 import synth  # noqa: E402
from paper_2408_14302_b200.signal_io import decimate_device  # noqa: E402

x = torch.from_numpy(synth.make_batch(2, clips=64)).cuda()
sc = synth.config_scales(2)
for aa in (False, True):
    for _ in range(2):
        d = decimate_device(x, 64, aa)
p = wh.CwthPlan(sc, None, 64, 160000, wavelet="rmor", output="log1p", norm="render", max_clips=64)
for _ in range(2):
    o = p.execute(x)
p = wh.CwthPlan(sc, None, 100, 160000, wavelet="rmor", output="log1p", max_clips=64, engine="simt")
for _ in range(2):
    o = p.execute(x)
torch.cuda.synchronize()
print("ok")
