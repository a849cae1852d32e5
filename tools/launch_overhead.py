"""Diagnostics: c2 kernel time with the bench's 256 MiB L2 flush (a torch fill kernel)
between launches vs back-to-back launches vs flush through a kernel that keeps the SM's
shared-memory carve-out (not used by bench.py; explains the gap between event time and
CTA lifetime)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_14302_b200 as wh  # noqa: E402
from paper_2408_14302_b200 import synth  # noqa: E402

x = torch.from_numpy(synth.make_batch(2, clips=64)).cuda()
plan = wh.CwthPlan(synth.config_scales(2), None, 64, 160000, wavelet="rmor", output="log1p", max_clips=64)
out = plan.execute(x)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def timed(pre):
    ts = []
    for _ in range(30):
        pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.execute(x, out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts) * 1e3


print(f"flush between (bench): {timed(lambda: flush.zero_()):.1f} us")
print(f"back to back:          {timed(lambda: None):.1f} us")
print(f"previous = same kernel (warm L2): {timed(lambda: plan.execute(x, out)):.1f} us")
