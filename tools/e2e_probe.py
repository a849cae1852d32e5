"""e2e (pinned host -> device -> host) time of c2 through CwthPlan.execute_host, for chunk-count experiments."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_14302_b200 as wh  # noqa: E402

w = bench.workload(sys.argv[1] if len(sys.argv) > 1 else "c2")
clips = w["clips"] if w["scaling"] == "weak" else 148
xh = bench.make_inputs(w, clips, 0)
plan = wh.CwthPlan(w["scales"], wh.MorletParams(), w["hop"], w["n"], wavelet=w["wavelet"], output=w["output"],
                   norm=w["norm"], max_clips=clips, engine="umma")
xpin = torch.from_numpy(xh).pin_memory()
opin = torch.empty((clips, len(w["scales"]), plan.frames), dtype=torch.float32).pin_memory()
xn, on = xpin.numpy(), opin.numpy()
for _ in range(3):
    plan.execute_host(xn, on)
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    plan.execute_host(xn, on)
    ts.append(time.perf_counter() - t0)
ts.sort()
print(f"{w['name']} e2e chunks={os.environ.get('WH_HOST_CHUNKS', 'default')}: median {ts[5] * 1e3:.3f} ms min {ts[0] * 1e3:.3f} ms"
      f" ({(xh.nbytes + on.nbytes) / ts[0] / 1e9:.1f} GB/s H2D+D2H)")
