"""Kernel time of c4-shaped batches at hops the panel-streaming path serves by default (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_14302_b200 as wh  # noqa: E402

w = bench.workload("c4h256")
x = torch.from_numpy(bench.make_inputs(w, w["clips"], 0)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for hop in [int(h) for h in sys.argv[1:]] or [320, 448, 576, 1088]:
    plan = wh.CwthPlan(w["scales"], wh.MorletParams(), hop, w["n"], wavelet=w["wavelet"], output=w["output"],
                       norm=w["norm"], max_clips=w["clips"], engine="umma")
    out = plan.execute(x)
    ts = []
    for i in range(23):
        flush.fill_(i & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.execute(x, out)
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    plan.close()
    print(f"hop {hop}: median {ts[len(ts) // 2]:.1f} us (TMA {'off' if os.environ.get('WH_UMMA_NO_TMA') else 'on'})", flush=True)
