"""Device timeline of one run_fused on a config (pinned host CSR), after
warm-up: every kernel and memcpy with start offset, duration and stream,
captured with torch.profiler (CUPTI activity records cover the library's own
launches).  Profiler overhead shifts host-side gaps; use it for overlap
structure, not for absolute wall time."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2008_03095_b200 as imx
from bench import pinned
from paper_2008_03095_b200 import configs

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
c = configs.CONFIGS[cfg]
g = configs.build(cfg)
host = imx.Graph(pinned(g.xadj), pinned(g.adj), pinned(g.weights), g.orig_ids)
del g
for i in range(4):
    gi = imx.Graph(host.xadj, host.adj, host.weights, host.orig_ids)
    run = imx.run_fused(gi, c.K, num_simulations=c.R, master_seed=0)
    _ = list(run.seeds)
    del run, gi
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    gi = imx.Graph(host.xadj, host.adj, host.weights, host.orig_ids)
    run = imx.run_fused(gi, c.K, num_simulations=c.R, master_seed=0)
    _ = list(run.seeds)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
min_us = float(sys.argv[2]) if len(sys.argv) > 2 else 50.0
print(f"{cfg}: {len(evs)} device activities; showing >= {min_us} us")
for e in evs:
    d = e.time_range.end - e.time_range.start
    if d >= min_us:
        print(f"{(e.time_range.start - t0) / 1e3:9.3f} ms  +{d / 1e3:8.3f} ms  {e.name[:90]}")
print("run.timings", {k: round(v * 1e3, 3) for k, v in run.timings.items()})
