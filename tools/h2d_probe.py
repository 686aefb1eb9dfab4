"""H2D bandwidth probe: pageable vs pinned, and host memcpy into pinned with
k threads (what a staged upload could reach)."""
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

def t(f, reps=20):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps

for mb in (4.4, 31, 256):
    n = int(mb * 1e6)
    src = np.random.randint(0, 255, n, dtype=np.uint8)
    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    pin = torch.empty(n, dtype=torch.uint8).pin_memory()
    pv = pin.numpy()
    s = torch.from_numpy(src)
    a = t(lambda: dst.copy_(s, non_blocking=False))
    b = t(lambda: dst.copy_(pin, non_blocking=True))
    c = t(lambda: np.copyto(pv, src))
    res = [f"{mb} MB: pageable {n/a/1e9:.1f} GB/s, pinned {n/b/1e9:.1f} GB/s, memcpy1 {n/c/1e9:.1f} GB/s"]
    for k in (2, 4, 8):
        ex = ThreadPoolExecutor(k)
        parts = np.array_split(np.arange(n), k)
        bounds = [(p[0], p[-1] + 1) for p in parts]
        def go():
            list(ex.map(lambda ab: np.copyto(pv[ab[0]:ab[1]], src[ab[0]:ab[1]]), bounds))
        d = t(go)
        res.append(f"memcpy{k} {n/d/1e9:.1f}")
        ex.shutdown()
    print(", ".join(res), flush=True)
import os
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
