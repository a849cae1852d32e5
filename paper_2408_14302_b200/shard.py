"""Clip sharding across GPUs.

Clips are independent, so a batch is split into contiguous clip ranges, one per rank
(or per device), with NO collective on the data path; every shard is computed by the
same plan on its own device and is byte-identical to the unsharded result.  The only
optional exchange is a gather of the scalograms onto one rank (NCCL all_gather /
gather via torch.distributed when multi-process, or peer copies when one process
drives several devices).

The reference has no multi-device code; its parallelism is a thread pool over rows
(wavelet.py:326-332) and over files (cli.py:193-206).
"""

from __future__ import annotations

import threading

import numpy as np


def shard_range(n_clips: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) clip range of ``rank`` out of ``world``."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("need 0 <= rank < world")
    if n_clips < 0:
        raise ValueError("n_clips must be >= 0")
    base, extra = divmod(n_clips, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def cwth_multi_device(x: np.ndarray, scales, params=None, hop: int = 128, *, devices=(0,),
                      wavelet: str = "cmor", output: str = "complex", norm=None,
                      engine: str = "auto") -> np.ndarray:
    """One process, one host thread per device: shard host clips [B, N] over ``devices``
    and return the host scalogram [B, S, F].  Each thread calls the C ABI (ctypes
    releases the GIL), so devices run concurrently."""
    from .wavelet import CwthPlan

    x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float32)
    B, n = x.shape
    devices = list(devices)
    ranges = [shard_range(B, len(devices), r) for r in range(len(devices))]
    # one plan per SHARD (a plan's staging buffers serve one host thread at a time, and the
    # same device may appear twice in ``devices``)
    plans = {r: CwthPlan(scales, params, hop, n, wavelet=wavelet, output=output, norm=norm,
                         max_clips=b - a, device=d, engine=engine)
             for r, (d, (a, b)) in enumerate(zip(devices, ranges)) if b > a}
    first = next(iter(plans.values()), None)
    frames = first.frames if first else -(-n // hop)
    dtype = first.out_dtype if first else (np.complex64 if output == "complex" else np.float32)
    out = np.empty((B, len(scales), frames), dtype=dtype)
    errors = []

    def run(r, a, b):
        try:
            plans[r].execute_host(x[a:b], out=out[a:b])
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=run, args=(r, a, b)) for r, (a, b) in enumerate(ranges) if b > a]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for p in plans.values():
        p.close()
    if errors:
        raise errors[0]
    return out


def gather_to_rank0(local, n_clips: int, group=None):
    """torch.distributed gather of per-rank scalogram shards [b_r, S, F] (contiguous clip
    ranges from :func:`shard_range`) into the full [n_clips, S, F] tensor on every rank
    (all_gather over padded shards; NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    sizes = [shard_range(n_clips, world, r) for r in range(world)]
    maxb = max(b - a for a, b in sizes)
    pad = torch.zeros((maxb,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([buf[: b - a] for buf, (a, b) in zip(bufs, sizes)], dim=0)
