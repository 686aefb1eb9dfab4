"""One-off parity check of the streamed host-CSR path at a width the tests do
not cover: C4 from a pinned host graph (chunked adjacency upload, pass 1 per
chunk, deferred speculation check) at R lanes (default 2048: two lane chunks
in the scan sampler), every lane against the oracle (oracle/scale_check.py)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_03095_b200 as imx
from bench import pinned
from oracle.scale_check import check_fused_run
from paper_2008_03095_b200 import configs

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
c = configs.CONFIGS[cfg]
g = configs.build(cfg)
host = imx.Graph(pinned(g.xadj), pinned(g.adj), pinned(g.weights), g.orig_ids)
g.drop_device()
t0 = time.perf_counter()
run = imx.run_fused(host, c.K, num_simulations=R, master_seed=0)
seeds = list(run.seeds)
print(f"{cfg} R={R}: run_fused {1e3 * (time.perf_counter() - t0):.1f} ms (first call), seeds {seeds[:5]}, "
      f"spread {run.spread:.3f}", flush=True)
rep = check_fused_run(run, host, c.K, R, 0, dense_window=4)
print(rep)
assert rep["ok"], rep
