"""Per-lane propagate cost vs. context width (is an L2-resident window faster?)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_03095_b200 as imx
from paper_2008_03095_b200 import configs
from paper_2008_03095_b200.context import DeviceContext

cfg = sys.argv[1]
widths = [int(w) for w in sys.argv[2].split(",")]
c = configs.CONFIGS[cfg]
g = configs.build(cfg)
X = imx.SimulationRandoms(c.R, 0).values
for w in widths:
    ctx = DeviceContext(g, X[:w], w)
    ctx.bench_propagate(2, flush_l2=True)
    r = ctx.bench_propagate(5, flush_l2=True)
    mb = g.n * w * 4 / 1e6
    print(f"{cfg} W={w:5d} L={mb:8.1f}MB total={r['total_ms']:.4f}ms per_lane_us={1e3 * r['total_ms'] / w:.3f} "
          f"init={r['init_ms']:.4f} hook={r['hook_ms']:.4f} compress={r['compress_ms']:.4f}")
    ctx.close()
