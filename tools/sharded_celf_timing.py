"""Wall time of the host-driven sharded CELF loop (celf.select_rounds) on one
context with LocalComm, vs the single-context persistent kernel: the per-round
host overhead a multi-rank run pays before any collective."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_03095_b200 as imx
from paper_2008_03095_b200 import configs
from paper_2008_03095_b200.celf import LocalComm, select_rounds
from paper_2008_03095_b200.context import DeviceContext

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = configs.CONFIGS[cfg]
g = configs.build(cfg)
X = imx.SimulationRandoms(c.R, 0).values
imx.build_hash_table(g).bind(g)
ctx = DeviceContext(g, X, c.R)
ctx.propagate()
gains = ctx.memoize(want_gains=True)
for rep in range(3):
    ctx.celf_reset(None)
    t0 = time.perf_counter()
    s1, g1, tr1 = ctx.celf_select(c.K)
    t1 = time.perf_counter()
    ctx.celf_reset(gains)
    t2 = time.perf_counter()
    s2, g2, tr2 = select_rounds(ctx, LocalComm(), c.K)
    t3 = time.perf_counter()
    same = s1.tolist() == s2.tolist() and np.array_equal(np.asarray(tr1), tr2)
    print(f"{cfg}: persistent kernel {1e3 * (t1 - t0):.2f} ms, host-driven rounds {1e3 * (t3 - t2):.2f} ms "
          f"({c.K} rounds, {len(tr2)} trace records), identical={same}")

if "--profile" in sys.argv:
    import cProfile
    import pstats
    ctx.celf_reset(gains)
    pr = cProfile.Profile()
    pr.enable()
    select_rounds(ctx, LocalComm(), c.K)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)
