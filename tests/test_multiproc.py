"""N>1 path on CPU: world_size-2 gloo process group exercising the clip sharding, the
optional gather and the max-over-ranks timing reduction that bench.py uses on GPUs.
The per-shard compute here is the CPU oracle (test infrastructure)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2408_14302_b200 import synth
from paper_2408_14302_b200.shard import gather_to_rank0, shard_range

N_CLIPS, N, HOP = 5, 3000, 32
SCALES = np.geomspace(1, 64, 10)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    from oracle import oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_range(N_CLIPS, world, rank)
    x = synth.make_batch(5, clips=b - a, n=N, start=a)
    local = O.cwth_batch(x, SCALES, HOP, wavelet="cmor", output="abs", norm="minmax", threads=1)
    full = gather_to_rank0(torch.from_numpy(local), N_CLIPS)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        np.save(os.path.join(outdir, "full.npy"), full.numpy())
        np.save(os.path.join(outdir, "tmax.npy"), t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_gather_is_bit_identical(tmp_path):
    from oracle import oracle as O

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    full = np.load(tmp_path / "full.npy")
    x = synth.make_batch(5, clips=N_CLIPS, n=N, start=0)
    ref = O.cwth_batch(x, SCALES, HOP, wavelet="cmor", output="abs", norm="minmax", threads=1)
    np.testing.assert_array_equal(full, ref)  # per-clip work is identical -> byte-equal
    assert float(np.load(tmp_path / "tmax.npy")[0]) == 2.0
