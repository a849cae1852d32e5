import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench, paper_2408_14302_b200 as wh
from oracle import oracle as O
w = bench.workload("c2")
x = torch.from_numpy(bench.make_inputs(w, 64, 0)).cuda()
T = np.array([2 * O.half_width(s) + 1 for s in w["scales"]], dtype=np.float64).sum()
for hop, eng in ((100, "simt"), (96, "umma"), (96, "simt"), (128, "umma"), (64, "simt"), (64, "umma")):
    plan = wh.CwthPlan(w["scales"], wh.MorletParams(), hop, w["n"], wavelet="rmor", output="log1p", max_clips=64, engine=eng)
    out = plan.execute(x)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(13):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); plan.execute(x, out); b.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(a.elapsed_time(b))
    ms = sorted(ts)[5]
    F = -(-w["n"] // hop)
    flops = 64 * F * T * 2
    print(f"hop {hop:4d} {eng}: {ms:.3f} ms  {64*128*F/ms/1e-3:.3e} coeffs/s  alg {flops/ms/1e9:.1f} TFLOP/s (SIMT folded executes half)", flush=True)
    plan.close()
