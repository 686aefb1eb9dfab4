"""Host wall time of each phase of run_fused's select on a config (after
warm-up), every phase fenced by a device synchronize."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2008_03095_b200 as imx
from bench import pinned
from paper_2008_03095_b200 import configs
from paper_2008_03095_b200.propagation import propagated_context
from paper_2008_03095_b200.selection import result_from_context

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
c = configs.CONFIGS[cfg]
g = configs.build(cfg)
host = imx.Graph(pinned(g.xadj), pinned(g.adj), pinned(g.weights), g.orig_ids)
del g
for it in range(4):
    gi = imx.Graph(host.xadj, host.adj, host.weights, host.orig_ids)
    marks = []

    def mark(name):
        torch.cuda.synchronize()
        marks.append((name, time.perf_counter()))

    mark("start")
    table = imx.build_hash_table(gi)
    randoms = imx.SimulationRandoms(c.R, 0)
    mark("graph")
    ctx, _ = propagated_context(gi, table, randoms.values, c.R, fuse_memo=True)
    mark("propagate")
    ctx.memoize(want_gains=False)
    mark("memoize")
    ctx.celf_reset(None)
    mark("celf_reset")
    seeds, gains, trace = ctx.celf_select(c.K)
    mark("celf_select")
    sel = result_from_context(ctx, seeds, gains, trace, c.R)
    _ = sel.spread
    mark("result")
    if it == 3:
        print(cfg, " ".join(f"{marks[i][0]}={1e3 * (marks[i][1] - marks[i - 1][1]):.2f}" for i in range(1, len(marks))),
              f"total={1e3 * (marks[-1][1] - marks[0][1]):.2f} ms", ctx.timings())
    del sel, ctx, table, gi
