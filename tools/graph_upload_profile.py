"""Phase times of the host-CSR graph upload (imx_graph_from_csr) on a config
(IMX_GRAPH_PROFILE marks) and the plain wall time without marks."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_03095_b200 as imx
from paper_2008_03095_b200 import configs

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
g = configs.build(cfg)
for i in range(6):
    gi = imx.Graph(g.xadj, g.adj, g.weights, g.orig_ids)
    if i == 5:
        os.environ["IMX_GRAPH_PROFILE"] = "1"
    t = time.perf_counter()
    gi.device_graph()
    dt = time.perf_counter() - t
    print(f"upload {i}: {dt * 1e3:.3f} ms", file=sys.stderr, flush=True)
    del gi
