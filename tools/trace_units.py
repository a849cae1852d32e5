"""CTA-0 timeline of the UMMA kernel (diagnostics): per unit, when each role starts/ends."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
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
plan.trace(True)
plan.execute(x, out)
torch.cuda.synchronize()
t = plan.trace(False)
t0 = t[t > 0].min()
names = ["mma_wait_win", "mma_start", "mma_end", "cv_start", "cv_stg|exp_ok", "cv_wempty|ex0", "cv_wok|ex1",
         "cv_done", "epi_wait", "epi_start", "epi_end"]
print("unit " + " ".join(f"{n:>13s}" for n in names) + "   (kcycles from first event)")
for u in range(12):
    if t[1, u] == 0:
        break
    print(f"{u:4d} " + " ".join(f"{(t[e, u] - t0) / 1e3:13.1f}" for e in range(len(names))))

# per-CTA entry/exit (globaltimer ns) of the traced launch
plan.trace(True)
t0ev = torch.cuda.Event(enable_timing=True)
t1ev = torch.cuda.Event(enable_timing=True)
t0ev.record()
plan.execute(x, out)
t1ev.record()
torch.cuda.synchronize()
tt, c = plan.trace(False, per_cta=True)
cyc = tt[14, 1] - tt[14, 0]
ns = c[0, 1] - c[0, 0]
print(f"CTA 0: {cyc} cycles in {ns} ns -> {cyc / ns * 1e3:.0f} MHz")
c = c[(c[:, 0] > 0)]
base = c[:, 0].min()
print(f"launch (events) {t0ev.elapsed_time(t1ev) * 1e3:.1f} us; CTAs {len(c)}: entry spread {(c[:, 0].max() - base) / 1e3:.1f} us, "
      f"exit min {(c[:, 1].min() - base) / 1e3:.1f} us median {(np.median(c[:, 1]) - base) / 1e3:.1f} us max {(c[:, 1].max() - base) / 1e3:.1f} us")
