"""Panel timeline of CTA 0's second unit on the tf32 panel-streaming path (diagnostics build)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_14302_b200 as wh  # noqa: E402

w = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "c4h1024")
clips = w["clips"]
x = torch.from_numpy(bench.make_inputs(w, clips, 0)).cuda()
plan = wh.CwthPlan(w["scales"], wh.MorletParams(), w["hop"], w["n"], wavelet=w["wavelet"], output=w["output"],
                   norm=w["norm"], max_clips=clips, engine="umma")
out = plan.execute(x)
plan.trace(True)
plan.execute(x, out)
torch.cuda.synchronize()
t = plan.trace(False)
ev = {4: "landed", 5: "converted", 6: "barrier", 12: "slot_free", 13: "fetched"}
t0 = t[4, 0]
print("panel " + " ".join(f"{n:>10s}" for n in ev.values()) + "  (cycles from the unit's first panel)")
for p in range(32):
    if t[4, p] == 0:
        break
    print(f"{p:5d} " + " ".join(f"{int(t[e, p] - t0):10d}" for e in ev))
