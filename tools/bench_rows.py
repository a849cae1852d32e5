"""Measurements for the SURVEY §8f rows (one B200): device-timed throughput of
decimate + cwth_decimate, the fused render plan vs the plain plan, and the batched scan
driver end to end (WAV decode -> GPU -> SCG1/PGM files) against the per-file CPU path of the
oracle port.  Prints one JSON object (copied into profiles/ by hand)."""
import json
import os
import statistics
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_14302_b200 as wh  # noqa: E402
from paper_2408_14302_b200 import cli, synth, wavio  # noqa: E402
from oracle import oracle as O  # noqa: E402


def dev_time(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


res = {}
# ---- cwth_decimate: 64 c2 clips, hop 64, anti-aliased, 128 scales 1-32 on the 250 Hz grid --
x = torch.from_numpy(synth.make_batch(2, clips=64)).cuda()
sc = np.geomspace(1.0, 32.0, 128)
dec_ms = dev_time(lambda: wh.decimate_device(x, 64, True))
dec = wh.decimate_device(x, 64, True)
plan = wh.CwthPlan(sc, None, 1, dec.shape[1], wavelet="rmor", output="log1p", max_clips=64)
out = plan.execute(dec)
cwt_ms = dev_time(lambda: plan.execute(dec, out))
coeffs = 64 * 128 * dec.shape[1]
res["cwth_decimate_c2_h64_aa"] = {"decimate_ms": dec_ms, "transform_ms": cwt_ms,
                                  "coeffs_per_s": coeffs / ((dec_ms + cwt_ms) / 1e3),
                                  "input_GBs_decimate": 64 * 160000 * 4 / (dec_ms / 1e3) / 1e9}
# ---- fused render vs plain magnitude (c2 workload) ------------------------------------------
w_sc = synth.config_scales(2)
p_plain = wh.CwthPlan(w_sc, None, 64, 160000, wavelet="rmor", output="log1p", max_clips=64)
p_rend = wh.CwthPlan(w_sc, None, 64, 160000, wavelet="rmor", output="log1p", norm="render", max_clips=64)
o1, o2 = p_plain.execute(x), p_rend.execute(x)
res["render_fused_c2"] = {"plain_ms": dev_time(lambda: p_plain.execute(x, o1)),
                          "render_u8_ms": dev_time(lambda: p_rend.execute(x, o2))}
# ---- scan driver end to end ------------------------------------------------------------------
with tempfile.TemporaryDirectory() as td:
    src = os.path.join(td, "in")
    os.makedirs(src)
    clips = synth.make_batch(2, clips=64)
    for i in range(64):
        wavio.write_wav(wh.SignalBuffer(clips[i].astype(np.float64) / max(1.0, np.abs(clips[i]).max()), 16000.0),
                        os.path.join(src, f"m{i:03d}.wav"), encoding="float32")
    argv = ["scan", src, "--out-dir", os.path.join(td, "out"), "--hop", "64", "--scales", "128",
            "--threads", "16"]
    cli.run_cli(argv)  # warm-up (plans, JIT of nothing)
    t0 = time.perf_counter()
    rc = cli.run_cli(argv)
    scan_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    rc2 = cli.run_cli(argv + ["--pgm"])
    scan_pgm_s = time.perf_counter() - t0
    # CPU per-file path (oracle port of the reference's process(): read, transform, write)
    from paper_2408_14302_b200 import scalogram as S
    grid = wh.make_scale_grid(20.0, 0.45 * 16000.0, 128, 16000.0)
    t0 = time.perf_counter()
    for i in range(4):
        sig = wavio.read_wav(os.path.join(src, f"m{i:03d}.wav"))
        v = O.cwth_batch(sig.samples.astype(np.float32), grid.scales, 64, threads=len(os.sched_getaffinity(0)))
        S.write_matrix_bin_raw(v.astype(np.complex64), 64, 16000.0, grid.scales, os.path.join(td, "cpu.scg1"))
    cpu_per_file = (time.perf_counter() - t0) / 4
    res["scan_64_files_160k_h64_128scales"] = {
        "rc": [rc, rc2], "gpu_scan_s": scan_s, "gpu_scan_pgm_s": scan_pgm_s,
        "files_per_s": 64 / scan_s, "cpu_port_s_per_file": cpu_per_file,
        "cpu_threads": len(os.sched_getaffinity(0)),
        "speedup_vs_cpu_port": cpu_per_file * 64 / scan_s}
print(json.dumps(res, indent=1))
