"""Diagnostics: launch list of the fused render plan vs plain / minmax plans (c2 shapes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_14302_b200 as wh  # noqa: E402
from paper_2408_14302_b200 import synth  # noqa: E402

x = torch.from_numpy(synth.make_batch(2, clips=64)).cuda()
sc = synth.config_scales(2)
for norm in (None, "minmax", "render"):
    p = wh.CwthPlan(sc, None, 64, 160000, wavelet="rmor", output="log1p", norm=norm, max_clips=64)
    o = p.execute(x)
    for _ in range(2):
        p.execute(x, o)
torch.cuda.synchronize()
