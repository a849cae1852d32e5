"""A/B kernel time of two builds of the library: python tools/ab.py LIB.so [config] (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_14302_b200 import _lib  # noqa: E402

_lib.load(os.path.abspath(sys.argv[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_14302_b200 as wh  # noqa: E402

w = bench.workload(sys.argv[2] if len(sys.argv) > 2 else "c2")
clips = w["clips"] if w["scaling"] == "weak" else 148
x = torch.from_numpy(bench.make_inputs(w, clips, 0)).cuda()
plan = wh.CwthPlan(w["scales"], wh.MorletParams(), w["hop"], w["n"], wavelet=w["wavelet"], output=w["output"],
                   norm=w["norm"], max_clips=clips, engine="umma")
out = plan.execute(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(43):
    flush.fill_(i & 255)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if os.environ.get("AB_SLEEP"):
        torch.cuda._sleep(2_000_000)  # the host enqueues the kernel before the GPU reaches the event
    a.record()
    plan.execute(x, out)
    b.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
print(f"{os.path.basename(sys.argv[1])} {w['name']}: median {ts[len(ts) // 2]:.1f} us min {ts[0]:.1f} us", flush=True)
