"""Time evaluate_seeds / sampling_cdf on the device against the C oracle.

    python tools/eval_timing.py [--configs c2,c3] [--r-eval 100000]

Worlds/s of the device path (wall clock around the public call, graph
resident, results copied back) vs. the OpenMP C oracle on all host cores
over a bounded sample of worlds; plus sampling_cdf wall time at the
config's R.  Prints one JSON line per config.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c3")
    ap.add_argument("--r-eval", type=int, default=100_000)
    ap.add_argument("--oracle-worlds", type=int, default=2000)
    args = ap.parse_args()
    import oracle
    import paper_2008_03095_b200 as imx
    from paper_2008_03095_b200 import configs
    from paper_2008_03095_b200.evaluation import evaluate_counts
    for name in args.configs.split(","):
        c = configs.CONFIGS[name]
        g = configs.build(name)
        seeds = np.random.default_rng(0).choice(g.n, size=c.K, replace=False)
        evaluate_counts(g, seeds, 4096, 1)                      # warm-up
        t = time.perf_counter()
        counts = evaluate_counts(g, seeds, args.r_eval, 1)
        dev_s = time.perf_counter() - t
        nw = min(args.oracle_worlds, args.r_eval)
        t = time.perf_counter()
        want = oracle.evaluate_counts(g.xadj, g.adj, g.weights, seeds, nw, 1)
        orc_s = time.perf_counter() - t
        assert np.array_equal(counts[:nw], want)
        randoms = imx.SimulationRandoms(c.R, 0)
        table = imx.build_hash_table(g)
        imx.sampling_cdf(g, table, randoms)
        t = time.perf_counter()
        res = imx.sampling_cdf(g, table, randoms)
        cdf_s = time.perf_counter() - t
        print(json.dumps(dict(
            config=name, n=g.n, edges=g.num_undirected_edges, k=len(seeds), r_eval=args.r_eval,
            device_s=round(dev_s, 4), device_worlds_per_s=round(args.r_eval / dev_s, 1),
            device_edge_draws_per_s=float(f"{args.r_eval * g.num_undirected_edges / dev_s:.4g}"),
            oracle_worlds=nw, oracle_threads=oracle.threads(), oracle_s=round(orc_s, 3),
            oracle_worlds_per_s=round(nw / orc_s, 1), speedup=round((args.r_eval / dev_s) / (nw / orc_s), 1),
            mean=float(counts.mean()), cdf_values=res.num_values, cdf_ks=res.ks_distance,
            cdf_s=round(cdf_s, 4))), flush=True)


if __name__ == "__main__":
    main()
