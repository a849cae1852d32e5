"""Parity + kernel time of the panel-streaming paths (fp16 / tf32) at large hops (diagnostics)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_14302_b200 as wh  # noqa: E402
from paper_2408_14302_b200 import synth  # noqa: E402
from oracle import oracle as O  # noqa: E402


def row_rel_err(got, ref):
    den = np.abs(ref).max(axis=-1, keepdims=True)
    den = np.where(den > 0, den, 1.0)
    return float((np.abs(got - ref) / den).max())


def parity(hop, n=60000, clips=3):
    x = synth.make_batch(4, clips=clips, n=n, start=2)
    sc = synth.config_scales(4)
    plan = wh.CwthPlan(sc, None, hop, n, wavelet="rmor", output="abs", max_clips=clips, engine="umma")
    got = plan.execute_host(x)
    plan.close()
    ref = O.cwth_batch(x, sc, hop, wavelet="rmor", output="abs")
    return row_rel_err(got, ref)


def timing(cfg):
    w = bench.workload(cfg)
    clips = w["clips"]
    x = torch.from_numpy(bench.make_inputs(w, clips, 0)).cuda()
    plan = wh.CwthPlan(w["scales"], wh.MorletParams(), w["hop"], w["n"], wavelet=w["wavelet"], output=w["output"],
                       norm=w["norm"], max_clips=clips, engine="umma")
    out = plan.execute(x)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
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
    # sampled parity of the full-size launch
    got = out[:2].cpu().numpy()
    ref = O.cwth_batch(x[:2].cpu().numpy(), np.asarray(w["scales"]), w["hop"], wavelet=w["wavelet"], output=w["output"])
    plan.close()
    return ts[len(ts) // 2], ts[0], row_rel_err(got, ref)


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "all"
    tag = f"PSTREAM={os.environ.get('WH_UMMA_PSTREAM')} TF32={os.environ.get('WH_UMMA_TF32')}"
    if mode in ("all", "parity"):
        for hop in (256, 320, 512, 1024, 2048):
            try:
                print(f"[{tag}] parity hop {hop}: row_rel_err {parity(hop):.3e}", flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"[{tag}] parity hop {hop}: FAILED {e}", flush=True)
    if mode in ("all", "time"):
        for cfg in sys.argv[2:] or ("c4h256", "c4h1024"):
            med, mn, err = timing(cfg)
            print(f"[{tag}] {cfg}: median {med:.1f} us min {mn:.1f} us  err {err:.3e}", flush=True)
