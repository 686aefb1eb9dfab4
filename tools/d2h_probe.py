"""Pinned/pageable D2H and H2D bandwidth of 91 MB (the C4 trace) on this box."""
import time
import torch
n = 91 * (1 << 20) // 8
d = torch.empty(n, dtype=torch.int64, device="cuda")
for pin in (True, False):
    h = torch.empty(n, dtype=torch.int64, pin_memory=pin)
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"D2H pinned={pin}: {dt * 1e3:.2f} ms = {n * 8 / dt / 1e9:.1f} GB/s")
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"H2D pinned={pin}: {dt * 1e3:.2f} ms = {n * 8 / dt / 1e9:.1f} GB/s")
