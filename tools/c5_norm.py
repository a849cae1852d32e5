"""c5 at full size: main kernel alone (norm=None) vs with per-clip min-max (reset + kernel + apply)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_14302_b200 as wh  # noqa: E402

w = bench.workload("c5")
clips = int(sys.argv[1]) if len(sys.argv) > 1 else w["clips"]
x = torch.from_numpy(bench.make_inputs(w, clips, 0)).cuda()
plans = {n: wh.CwthPlan(w["scales"], wh.MorletParams(), w["hop"], w["n"], wavelet=w["wavelet"], output=w["output"],
                        norm=n, max_clips=clips, engine="umma") for n in (None, "minmax")}
out = torch.empty((clips, len(w["scales"]), plans[None].frames), dtype=torch.float32, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
res = {None: [], "minmax": []}
for it in range(4):
    for n, p in plans.items():
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        p.execute(x, out)
        b.record()
        torch.cuda.synchronize()
        if it:
            res[n].append(a.elapsed_time(b))
for n, v in res.items():
    print(f"c5 {clips} clips norm={n}: {sorted(v)} ms", flush=True)
