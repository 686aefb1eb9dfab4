"""Pinned host->device copy bandwidth with 1, 2 and 4 concurrent streams."""
import time
import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4, 1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        t0 = time.perf_counter()
        per = n // ns
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * per:(i + 1) * per].copy_(h[i * per:(i + 1) * per], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"streams {ns}: {n / best / 1e9:.1f} GB/s")
