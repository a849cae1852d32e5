#!/usr/bin/env python
"""bench.py -- CWTH scalogram coefficients/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One "step" = one pass of the hot path (cwth_batch with the config's fused epilogue) over
the rank's batch of synthetic clips.  Default workload: BASELINE config 2 (configs[1]):
64 clips x 160,000 fp32 samples of synthetic machine noise per GPU, real Morlet, 128
geometric scales 1-128, hop 64, log1p(|W|).  N>1 (torchrun, one process per GPU): every
rank processes its own 64 clips -- clips are independent, no data-path collective
(weak scaling).  ``--config c5`` runs config 5 (4096 clips split across ranks, strong
scaling).

Printed JSON (rank 0, one line): value = coeffs/s of the whole job from CUDA-event kernel
time with inputs resident in HBM (L2 flushed by a 256 MiB write before every step);
e2e = the same metric through the public API with pinned HOST buffers (H2D + kernels +
D2H inside the timed region); roofline = the main kernel against its binding roof:
algorithmic FLOP/s vs the measured bf16 tensor peak, or algorithmic bytes/s vs the measured
HBM bandwidth, whichever bounds the algorithm (c2: HBM); cpu_baseline = the oracle port (oracle/) on the box's
host cores, on the same clips.  ``--impl reference`` times only the CPU reference port.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_2408_14302_b200 import synth  # noqa: E402

METRIC = "CWTH scalogram coeffs/sec (clips x scales x frames)"
UNIT = "coeffs/s"
L2_FLUSH_BYTES = 256 << 20


def workload(name: str):
    """Config name -> dict(cfg_id, clips(total), n, scales, hop, wavelet, output, norm, scaling)."""
    base = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5}
    hop_override = None
    key = name
    if name.startswith("c4h"):
        key, hop_override = "c4", int(name[3:])
    cid = base[key]
    cfg = dict(synth.CONFIGS[cid])
    w = dict(cfg_id=cid, name=name, clips=cfg["clips"], n=cfg["n"],
             scales=synth.config_scales(cid), hop=hop_override or cfg["hop"],
             wavelet=cfg["wavelet"], output=cfg["output"], norm=cfg["norm"],
             scaling="strong" if cid == 5 else "weak")
    return w


def alg_flops(w, clips: int) -> float:
    """unfolded direct correlation, 2*T (real) or 4*T (complex) flop/coeff."""
    from oracle import oracle as O  # only for the integer half widths (same fp64 formula)

    F = -(-w["n"] // w["hop"])
    T = np.array([2 * O.half_width(s) + 1 for s in w["scales"]], dtype=np.float64)
    per = 2.0 if w["wavelet"] == "rmor" else 4.0
    return float(clips) * F * per * T.sum()


def coeffs(w, clips: int) -> float:
    return float(clips) * len(w["scales"]) * (-(-w["n"] // w["hop"]))


def make_inputs(w, clips: int, start: int) -> np.ndarray:
    return synth.make_batch(w["cfg_id"], clips=clips, n=w["n"], start=start)


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d["bf16_tflops"], d.get("bf16_tflops_sustained"), d["hbm_gbs"], "measured"
    except Exception:  # noqa: BLE001
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.proc, self.lines = device, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def wait_first(self, timeout=5.0):
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.02)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_reference(w, x: np.ndarray, threads: int):
    """Time the CPU port of the reference (oracle/) on clips x: returns seconds."""
    from oracle import oracle as O

    t0 = time.perf_counter()
    if w["hop"] == 1:
        # the reference routes hop = 1 rows to its FFT path (wavelet.py:249,257); the
        # per-clip routed port runs clips in a thread pool (the C kernel drops the GIL)
        from concurrent.futures import ThreadPoolExecutor

        def one(c):
            v = O.cwth_strided_routed(x[c], w["scales"], w["hop"])
            return O.epilogue(v, w["wavelet"], w["output"], w["norm"])

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, range(x.shape[0])))
    else:
        O.cwth_batch(x, w["scales"], w["hop"], wavelet=w["wavelet"], output=w["output"],
                     norm=w["norm"], threads=threads)
    return time.perf_counter() - t0


def run_reference(args, w):
    """--impl reference: the reference's CPU path (oracle port) on the host cores."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    sample = min(args.ref_clips, w["clips"])
    x = make_inputs(w, sample, 0)
    for _ in range(max(args.warmup, 1)):
        cpu_reference(w, x[: min(4, sample)], threads)
    times = [cpu_reference(w, x, threads) for _ in range(args.steps)]
    t = sum(times)
    value = coeffs(w, sample) * args.steps / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": w["scaling"], "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded MIMII stand-in, SURVEY.md §8d)",
        # the same keys as the GPU arm's config; a step is `sample` clips (the whole per-GPU
        # batch for c2) on the host cores
        "config": {"workload": w["name"], "clips_per_gpu": sample, "n_samples": w["n"],
                   "scales": len(w["scales"]), "scale_range": [float(w["scales"][0]),
                                                              float(w["scales"][-1])],
                   "hop": w["hop"], "wavelet": w["wavelet"], "output": w["output"],
                   "norm": w["norm"], "engine": "cpu-oracle-port", "parallelism": f"host threads x{threads}",
                   "l2": "n/a (host)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{sample} clips of {w['name']} per step, oracle/wh_oracle.c "
                                   f"folded f64 kernel (numba-equivalent), {threads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, w):
    import torch

    world, rank, local = dist_setup()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2408_14302_b200 as wh

    # shard: weak scaling keeps the per-rank batch; strong scaling splits the total
    if w["scaling"] == "weak":
        per_rank = args.clips or w["clips"]
        start = rank * per_rank
    else:
        from paper_2408_14302_b200.shard import shard_range

        total = args.clips or w["clips"]
        start, stop = shard_range(total, world, rank)
        per_rank = stop - start
    xh = make_inputs(w, per_rank, start)
    params = wh.MorletParams()
    plan = wh.CwthPlan(w["scales"], params, w["hop"], w["n"], wavelet=w["wavelet"],
                       output=w["output"], norm=w["norm"], max_clips=per_rank, device=local,
                       engine=args.engine)
    x = torch.from_numpy(xh).to(dev)
    out_dtype = torch.complex64 if w["output"] == "complex" else torch.float32
    out = torch.empty((per_rank, len(w["scales"]), plan.frames), dtype=out_dtype, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    # ---- device-resident timed region -------------------------------------------------
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            flush.zero_()
            plan.execute(x, out, stream=stream)
    barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        clk.wait_first()
        barrier()
        n0 = len(clk.lines)
        with torch.cuda.stream(stream):
            for s, e in evs:
                flush.zero_()
                s.record(stream)
                plan.execute(x, out, stream=stream)
                e.record(stream)
        barrier()
        # keep the same load running (untimed) until the sampler has seen it a few
        # times, so the clock record describes the GPU under this workload
        t0 = time.time()
        while len(clk.lines) < n0 + 4 and time.time() - t0 < 2.0:
            with torch.cuda.stream(stream):
                for _ in range(8):
                    flush.zero_()
                    plan.execute(x, out, stream=stream)
            torch.cuda.synchronize(dev)
    dev_ms = sum(s.elapsed_time(e) for s, e in evs)
    # ---- end-to-end through the public API with pinned host buffers ------------------
    e2e_ms = None
    if not args.no_e2e:
        xpin = torch.from_numpy(xh).pin_memory()
        opin = torch.empty(tuple(out.shape), dtype=out_dtype).pin_memory()
        xnp, onp = xpin.numpy(), opin.numpy()
        for _ in range(max(1, min(args.warmup, 3))):
            plan.execute_host(xnp, onp)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            plan.execute_host(xnp, onp)
        e2e_ms = 1e3 * (time.perf_counter() - t0)
        barrier()
    # ---- reduce over ranks --------------------------------------------------------------
    vals = torch.tensor([dev_ms, e2e_ms or 0.0], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(vals, op=torch.distributed.ReduceOp.MAX)
    dev_ms, e2e_ms_max = float(vals[0]), float(vals[1])
    total_clips = per_rank * world if w["scaling"] == "weak" else (args.clips or w["clips"])
    value = coeffs(w, total_clips) * args.steps / (dev_ms / 1e3)
    result = None
    if rank == 0:
        bf16, bf16_sus, hbm, peak_kind = peaks()
        # main-kernel time: with min-max normalisation the plan also launches the
        # reset/normalise kernels; time the main kernel alone through a norm=None plan
        kern_ms = dev_ms / args.steps
        if w["norm"] is not None:
            plan2 = wh.CwthPlan(w["scales"], params, w["hop"], w["n"], wavelet=w["wavelet"],
                                output=w["output"], norm=None, max_clips=per_rank, device=local,
                                engine=args.engine)
            with torch.cuda.stream(stream):
                plan2.execute(x, out, stream=stream)
                ks = []
                for _ in range(min(args.steps, 5)):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    plan2.execute(x, out, stream=stream)
                    b.record(stream)
                    ks.append((a, b))
            torch.cuda.synchronize(dev)
            kern_ms = statistics.median(a.elapsed_time(b) for a, b in ks)
            plan2.close()
        flops = alg_flops(w, per_rank)
        achieved = flops / (kern_ms / 1e3) / 1e12
        traffic = None
        tpath = os.path.join(REPO, "profiles", "traffic.json")
        if os.path.exists(tpath):
            with open(tpath) as f:
                traffic = json.load(f).get(f"{w['name']}:{plan.engine}:{per_rank}")
        in_bytes = 4.0 * per_rank * w["n"]
        out_bytes = float(out.numel() * out.element_size())
        # The binding roof of the algorithm: algorithmic flops against the
        # measured bf16 tensor peak, or algorithmic bytes (input once + output once) against
        # the measured HBM copy bandwidth -- whichever lower bound on the kernel time is
        # larger.  c2 (92 flop/B) sits below the ridge (1630e12 / 6547.5e9 = 249 flop/B): HBM.
        alg_bytes = in_bytes + out_bytes
        t_tensor, t_hbm = flops / (bf16 * 1e12), alg_bytes / (hbm * 1e9)
        kern_s = kern_ms / 1e3
        common = {"traffic": traffic, "kernel": "k_umma" if plan.engine == "umma" else "k_simt",
                  "kernel_ms": kern_ms, "alg_flops_per_launch": flops,
                  "alg_bytes_per_launch": alg_bytes,
                  "tensor_view": {"achieved_tflops": achieved, "peak_tflops": bf16,
                                  "frac": achieved / bf16,
                                  "note": "split-fp16 x3 products: executed MMA flops ~3x "
                                          "algorithmic (minus skipped tail cross terms) + K padding"},
                  "hbm_view": {"achieved_gbs": alg_bytes / kern_s / 1e9, "peak_gbs": hbm,
                               "frac": alg_bytes / kern_s / 1e9 / hbm},
                  "peak_source": f"{peak_kind} MEASURED_PEAKS.json burst figures (the kernel "
                                 f"is timed alone between L2 flushes)"}
        if t_hbm >= t_tensor:
            roofline = {"bound": "hbm", "achieved": alg_bytes / kern_s / 1e9, "peak": hbm,
                        "unit": "GB/s", "frac": alg_bytes / kern_s / 1e9 / hbm, **common}
        else:
            roofline = {"bound": "tensor", "achieved": achieved, "peak": bf16, "unit": "TFLOP/s",
                        "frac": achieved / bf16, **common}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            threads = len(os.sched_getaffinity(0))
            sample = min(per_rank, args.ref_clips)
            xs = xh[:sample]
            cpu_reference(w, xs[:2], threads)  # warm-up
            ts = [cpu_reference(w, xs, threads) for _ in range(3)]
            cpu = {"value": coeffs(w, sample) / statistics.median(ts), "unit": UNIT,
                   "cores": threads, "kind": "port",
                   "sample": f"{sample} clips of {w['name']} (the first clips of this workload), "
                             f"median of 3; oracle/wh_oracle.c folded f64 kernel with the "
                             f"reference's epilogue, {threads} threads"}
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": w["scaling"], "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded MIMII stand-in, SURVEY.md §8d)",
            "config": {"workload": w["name"], "clips_per_gpu": per_rank, "n_samples": w["n"],
                       "scales": len(w["scales"]), "scale_range": [float(w["scales"][0]),
                                                                  float(w["scales"][-1])],
                       "hop": w["hop"], "wavelet": w["wavelet"], "output": w["output"],
                       "norm": w["norm"], "engine": plan.engine, "parallelism": f"clip-shard x{world}",
                       "l2": "flushed: 256 MiB device write before every timed step"},
            "e2e": {"value": (coeffs(w, total_clips) * args.e2e_steps / (e2e_ms_max / 1e3))
                    if e2e_ms is not None else None,
                    "unit": UNIT, "h2d_bytes_per_step": int(in_bytes),
                    "d2h_bytes_per_step": int(out_bytes),
                    "note": "CwthPlan.execute_host -> wh_execute_host: pinned H2D + kernels + "
                            "D2H of the full scalogram, host wall clock, max over ranks"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "gpu_launches": plan.launches(per_rank) * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(result), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    plan.close()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2",
                    help="c1..c5 or c4h{1,16,64,256,1024} (default c2 = BASELINE configs[1])")
    ap.add_argument("--engine", choices=["auto", "simt", "umma"], default="auto")
    ap.add_argument("--clips", type=int, default=0, help="override clips per GPU (weak) / total (strong)")
    ap.add_argument("--ref-clips", type=int, default=64, help="clips in the CPU-baseline sample")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    w = workload(args.config)
    if args.impl == "reference":
        return run_reference(args, w)
    return run_ours(args, w)


if __name__ == "__main__":
    sys.exit(main())
