"""Time the reference's own Python run_fused (pipeline.py:44-66, imported
read-only from /root/reference) on C1 and C2 in THIS container, at
n_threads=1 and n_threads=os.cpu_count(), beside the oracle port (C/OpenMP)
on the same graph -- BASELINE.md section 4.2.  The reference cannot travel to
the GPU box; the log is committed under profiles/.

    PYTHONPATH=/root/reference/pkg/src python tools/reference_python_timing.py
"""
import json
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
import oracle                                     # noqa: E402
from infmax.graph import Graph as RefGraph        # noqa: E402
from infmax.pipeline import run_fused as ref_run_fused   # noqa: E402
from oracle.scale_check import config_host_graph  # noqa: E402
from paper_2008_03095_b200 import configs         # noqa: E402

out = []
for cfg in ("c1", "c2"):
    c = configs.CONFIGS[cfg]
    xadj, adj, w = config_host_graph(cfg)
    g = RefGraph(xadj=xadj, adj=adj, weights=w, orig_ids=np.arange(len(xadj) - 1, dtype=np.int64))
    for nt in (1, os.cpu_count()):
        t0 = time.perf_counter()
        run = ref_run_fused(g, c.K, num_simulations=c.R, master_seed=0, n_threads=nt)
        dt = time.perf_counter() - t0
        out.append({"config": cfg, "impl": "reference infmax.run_fused (Python/numpy)", "n_threads": nt,
                    "k_seed_wall_s": dt, "timings": {k: round(v, 4) for k, v in run.timings.items()},
                    "seeds_head": [int(s) for s in run.selection.seeds[:5]], "spread": run.selection.spread})
        print(json.dumps(out[-1]), flush=True)
    t0 = time.perf_counter()
    o = oracle.run_fused(xadj, adj, w, c.K, c.R, 0)
    dt = time.perf_counter() - t0
    assert o["seeds"].tolist() == [int(s) for s in run.selection.seeds]
    out.append({"config": cfg, "impl": "oracle port (C/OpenMP)", "n_threads": oracle.threads(),
                "k_seed_wall_s": dt, "seeds_match_reference": True})
    print(json.dumps(out[-1]), flush=True)
print(json.dumps({"host": platform.processor() or platform.machine(), "cpu_count": os.cpu_count(),
                  "numpy": np.__version__}))
