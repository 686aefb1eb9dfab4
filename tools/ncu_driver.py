"""Small driver for ncu: build a config graph, run propagate a few times."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_03095_b200 as imx
from paper_2008_03095_b200 import configs
from paper_2008_03095_b200.context import DeviceContext

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = configs.CONFIGS[cfg]
R = int(sys.argv[3]) if len(sys.argv) > 3 else c.R     # lane override (smaller label matrix for ncu)
g = configs.build(cfg)
X = imx.SimulationRandoms(R, 0).values
ctx = DeviceContext(g, X, R)
ctx.propagate()          # one-time per-graph setup (sampler index, heavy-row slices) outside the window
res = ctx.bench_propagate(reps, flush_l2=True)
ctx.memoize(want_gains=False)
from paper_2008_03095_b200.build import source_hash
print(cfg, res)
print(f"src_hash={source_hash()}")
