"""cProfile of one run_fused on a benchmark config (host-side breakdown)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_03095_b200 as imx
from paper_2008_03095_b200 import configs

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c2"
c = configs.CONFIGS[cfg]
g = configs.build(cfg)
if "--pinned" in sys.argv:
    from bench import pinned
    g = imx.Graph(pinned(g.xadj), pinned(g.adj), pinned(g.weights), g.orig_ids)
for _ in range(2):
    gi = imx.Graph(g.xadj, g.adj, g.weights, g.orig_ids)
    run = imx.run_fused(gi, c.K, c.R, 0)
gi = imx.Graph(g.xadj, g.adj, g.weights, g.orig_ids)
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
run = imx.run_fused(gi, c.K, c.R, 0)
pr.disable()
print("wall", time.perf_counter() - t0, "timings", run.timings)
print("ctx timings", run._ctx.timings())
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
