"""run_fused wall times, back to back, on a config with the host CSR in
pinned memory (what bench.py's e2e leg does), one line per step."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_03095_b200 as imx
from bench import pinned
from paper_2008_03095_b200 import configs

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
c = configs.CONFIGS[cfg]
g = configs.build(cfg)
host = imx.Graph(pinned(g.xadj), pinned(g.adj), pinned(g.weights), g.orig_ids)
del g
run = None
for i in range(steps):
    gi = imx.Graph(host.xadj, host.adj, host.weights, host.orig_ids)
    run = None
    t0 = time.perf_counter()
    run = imx.run_fused(gi, c.K, num_simulations=c.R, master_seed=0)
    s = list(run.seeds)
    dt = time.perf_counter() - t0
    print(f"{cfg} step {i}: {dt * 1e3:8.2f} ms  " + " ".join(f"{k}={v * 1e3:.1f}" for k, v in run.timings.items()), flush=True)
