"""Per-role wait breakdown of the UMMA kernel (diagnostics counters, wh_plan_profile)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_14302_b200 as wh  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--clips", type=int, default=0)
a = ap.parse_args()
w = bench.workload(a.config)
clips = a.clips or (w["clips"] if w["scaling"] == "weak" else 148)
x = torch.from_numpy(bench.make_inputs(w, clips, 0)).cuda()
plan = wh.CwthPlan(w["scales"], wh.MorletParams(), w["hop"], w["n"], wavelet=w["wavelet"],
                   output=w["output"], norm=w["norm"], max_clips=clips, engine="umma")
out = plan.execute(x)
plan.profile(True)
plan.execute(x, out)
torch.cuda.synchronize()
c = plan.profile(False)
warps = {"producer": 1, "mma": 0.5, "converter": 6, "epilogue": 8, "relay": 0.5}
names = {"producer": ["b_empty", "issue", "-"], "mma": ["win_full", "acc_empty", "b_full"],
         "converter": ["stg_full", "win_empty", "convert"], "epilogue": ["acc_full", "-", "-"],
         "relay": ["win_full", "-", "b_full"]}
sms = min(148, clips * ((plan.frames + 127) // 128))
for r, v in c.items():
    n = warps[r] * sms
    if v[3] == 0:
        continue
    tot = v[3] / n
    parts = ", ".join(f"{names[r][i]} {v[i] / n / tot * 100:5.1f}%" for i in range(3) if names[r][i] != "-")
    print(f"{w['name']} {r:9s} total {tot / 1e3:8.1f} kcyc  waits: {parts}")
