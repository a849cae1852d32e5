"""Kernel time of one config under WH_UMMA_DBG diagnostic bits (results invalid when bits set)."""
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
ap.add_argument("--bits", default="0,1,2,3,32,64,96,4,5,6,7")
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
w = bench.workload(a.config)
clips = a.clips or (w["clips"] if w["scaling"] == "weak" else 148)
x = torch.from_numpy(bench.make_inputs(w, clips, 0)).cuda()
plan = wh.CwthPlan(w["scales"], wh.MorletParams(), w["hop"], w["n"], wavelet=w["wavelet"],
                   output=w["output"], norm=w["norm"], max_clips=clips, engine="umma")
out = plan.execute(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for bits in [int(b) for b in a.bits.split(",")]:
    os.environ["WH_UMMA_DBG"] = str(bits)
    ts = []
    for i in range(a.iters + 3):
        flush.fill_(i & 255)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.execute(x, out)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"{a.config} dbg={bits:4d}: median {ts[len(ts) // 2]:8.1f} us  min {ts[0]:8.1f} us", flush=True)
os.environ.pop("WH_UMMA_DBG")
