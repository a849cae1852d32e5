"""c2 kernel time after different L2 flushes (torch zero_, fill kernel with default / max-smem carveout)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2408_14302_b200 as wh  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libflush_probe.so"))
lib.flush_fill.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_int, ctypes.c_void_p]
w = bench.workload("c2")
x = torch.from_numpy(bench.make_inputs(w, 64, 0)).cuda()
plan = wh.CwthPlan(w["scales"], wh.MorletParams(), w["hop"], w["n"], wavelet=w["wavelet"], output=w["output"],
                   max_clips=64, engine="umma")
out = plan.execute(x)
buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for mode in ("torch_zero", "fill_default", "fill_carve100", "torch_zero", "fill_carve100"):
    ts = []
    for i in range(33):
        if mode == "torch_zero":
            buf.zero_()
        else:
            lib.flush_fill(buf.data_ptr(), buf.numel(), i & 255, -1 if mode == "fill_default" else 100, st)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        plan.execute(x, out)
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    print(f"{mode:14s}: median {ts[len(ts) // 2]:.1f} us min {ts[0]:.1f} us", flush=True)
