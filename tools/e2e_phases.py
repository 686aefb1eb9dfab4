"""Host-side phase breakdown of run_fused on a config (pinned host CSR),
after warm-up: the library's own phase clocks (IMX_GRAPH_PROFILE,
IMX_CELF_PROFILE) plus run.timings and the context's device timings."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_03095_b200 as imx
from bench import pinned
from paper_2008_03095_b200 import configs

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = configs.CONFIGS[cfg]
g = configs.build(cfg)
host = imx.Graph(pinned(g.xadj), pinned(g.adj), pinned(g.weights), g.orig_ids)
for i in range(6):
    if i == 5 and os.environ.get("E2E_GRAPH_PROFILE"):
        os.environ["IMX_GRAPH_PROFILE"] = "1"      # its phase marks synchronise the graph stream
    gi = imx.Graph(host.xadj, host.adj, host.weights, host.orig_ids)
    t0 = time.perf_counter()
    run = imx.run_fused(gi, c.K, num_simulations=c.R, master_seed=0)
    s = list(run.seeds)
    dt = time.perf_counter() - t0
print(f"{cfg} wall {dt * 1e3:.3f} ms", {k: round(v * 1e3, 3) for k, v in run.timings.items()})
print("device", {k: (round(v, 3) if isinstance(v, float) else v) for k, v in run._ctx.timings().items()})
