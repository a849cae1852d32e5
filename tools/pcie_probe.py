import torch, time
d = torch.empty(82_000_000 // 4, device="cuda"); h = torch.empty(82_000_000 // 4).pin_memory()
hi = torch.empty(41_000_000 // 4).pin_memory(); di = torch.empty(41_000_000 // 4, device="cuda")
for name, fn in (("D2H 82MB", lambda: h.copy_(d, non_blocking=True)), ("H2D 41MB", lambda: di.copy_(hi, non_blocking=True))):
    for _ in range(3): fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10): fn()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 10
    print(name, f"{dt*1e3:.3f} ms", f"{(82e6 if 'D2H' in name else 41e6)/dt/1e9:.1f} GB/s")
