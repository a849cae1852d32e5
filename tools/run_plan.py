"""Run one config's plan a few times (small driver for ncu / compute-sanitizer)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_14302_b200 as wh  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--engine", default="auto")
ap.add_argument("--clips", type=int, default=0)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
w = bench.workload(a.config)
clips = a.clips or (w["clips"] if w["scaling"] == "weak" else 64)
x = torch.from_numpy(bench.make_inputs(w, clips, 0)).cuda()
plan = wh.CwthPlan(w["scales"], wh.MorletParams(), w["hop"], w["n"], wavelet=w["wavelet"],
                   output=w["output"], norm=w["norm"], max_clips=clips, engine=a.engine)
print("engine", plan.engine, flush=True)
for _ in range(a.iters):
    out = plan.execute(x)
torch.cuda.synchronize()
print("ok", float(out.float().abs().mean()))
