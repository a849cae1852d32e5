"""Parity (a few clips vs the oracle) + kernel time of one config under the current env (experiments)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_14302_b200 as wh  # noqa: E402
from oracle import oracle as O  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--clips", type=int, default=0)
ap.add_argument("--check", type=int, default=2)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
w = bench.workload(a.config)
clips = a.clips or (w["clips"] if w["scaling"] == "weak" else 148)
xs = bench.make_inputs(w, clips, 0)
x = torch.from_numpy(xs).cuda()
plan = wh.CwthPlan(w["scales"], wh.MorletParams(), w["hop"], w["n"], wavelet=w["wavelet"],
                   output=w["output"], norm=w["norm"], max_clips=clips, engine="umma")
out = plan.execute(x)
torch.cuda.synchronize()
if a.check:
    got = out[: a.check].cpu().numpy()
    ref = O.cwth_batch(xs[: a.check], w["scales"], w["hop"], wavelet=w["wavelet"], output=w["output"],
                       norm=w["norm"])
    if w["output"] == "log1p" or w["norm"]:
        err = float(np.abs(got - ref).max())
    else:
        err = float((np.abs(got - ref) / np.abs(ref).max(axis=-1, keepdims=True)).max())
    print(f"{a.config} parity over {a.check} clips: {err:.3e}", flush=True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
sweep = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
mode = os.environ.get("FLUSH", "write")
ts = []
for i in range(a.iters + 3):
    if mode in ("write", "write+read"):
        flush.fill_(i & 255)
    if mode == "write+read":
        float(sweep.view(torch.int32).sum())  # read sweep: the L2 ends full of clean lines
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.execute(x, out)
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1) * 1e3)
ts.sort()
print(f"{a.config} flush={mode} env V={os.environ.get('WH_UMMA_V', '-')}: median {ts[len(ts) // 2]:.1f} us min {ts[0]:.1f} us", flush=True)
