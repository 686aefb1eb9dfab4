"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture records the reference's own outputs (CSR, weights, hashes,
thresholds, X, labels, sizes, gains, seeds, trace, sigma, spread_se) for a
seeded input, so the oracle and the CUDA path can be pinned to them on any
machine.  Inputs: the reference's ER generator + weight schemes (as its tests
use them), hand-built known-answer graphs, and the C1/C2 benchmark graphs
from this repo's Chung-Lu generator (the reference has none).
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from infmax.graph import Graph, apply_weights, generate_er, parse_weight_scheme  # noqa: E402
from infmax.hashing import build_hash_table, slot_thresholds, SimulationRandoms  # noqa: E402
from infmax.pipeline import run_fused  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def record(name, g, edges, scheme, weight_seed, R, seed, k, full=True):
    run = run_fused(g, k, num_simulations=R, master_seed=seed)
    tr = np.array([(t.vertex, t.stale_gain, t.fresh_gain, int(t.committed), t.seeds_before)
                   for t in run.selection.trace], dtype=np.int64).reshape(-1, 5)
    out = dict(
        n=np.int64(g.n), edges=np.asarray(edges, np.int64).reshape(-1, 2),
        scheme=np.array(scheme), weight_seed=np.int64(weight_seed),
        xadj=g.xadj, adj=g.adj, weights=g.weights,
        hashes=build_hash_table(g).hashes, thr=slot_thresholds(g),
        X=run.randoms.values, R=np.int64(R), master_seed=np.int64(seed), k=np.int64(k),
        seeds=np.asarray(run.seeds, np.int64), seed_gains=np.asarray(run.selection.gains, np.int64),
        sigma=np.int64(run.selection.sigma), spread=np.float64(run.spread),
        spread_se=np.float64(run.spread_se), trace=tr,
        labels_sha=np.array(digest(run.labels.astype(np.int32))),
        sizes_sha=np.array(digest(np.ascontiguousarray(run.sizes).astype(np.int32))),
    )
    from infmax.propagation import component_sizes_and_gains
    _, gains = component_sizes_and_gains(run.labels, run.randoms.num_scored)
    out["gains"] = gains
    if full:
        out["labels"] = run.labels.astype(np.int32)
        out["sizes"] = np.ascontiguousarray(run.sizes).astype(np.int32)
    else:  # large inputs: keep digests of the derived arrays, edges as int32
        for key in ("xadj", "adj", "weights", "hashes", "thr"):
            out[key + "_sha"] = np.array(digest(out.pop(key)))
        out["edges"] = out["edges"].astype(np.int32)
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(f"{name}: n={g.n} m={g.m} R={R} k={k} seeds={list(run.seeds)[:8]} "
          f"trace={len(tr)} spread={run.spread:.4f}")


def weighted_er(n, deg, scheme, graph_seed, weight_seed):
    g0 = generate_er(n, deg, seed=graph_seed)
    canon = g0.canonical_slots
    edges = np.column_stack([g0.sources[canon], g0.adj[canon]])
    g = apply_weights(g0, parse_weight_scheme(scheme), rng_seed=weight_seed)
    return g, edges


def main():
    # known-answer graphs (weights 1 / mixed), tests/test_selection.py:34-58
    kat = {
        "kat_two_components": ([(0, 1), (1, 2), (0, 2), (3, 4)], 5, 1.0, 8, 0, 2),
        "kat_path3": ([(0, 1), (1, 2)], 3, 1.0, 8, 0, 3),
        "kat_ties": ([(0, 1), (2, 3)], 4, 1.0, 8, 0, 2),
        "kat_dead_middle": ([(0, 1), (1, 2)], 3, [1.0, 0.0], 16, 0, 2),
    }
    for name, (edges, n, w, R, seed, k) in kat.items():
        g = Graph.from_edges(n, edges, w)
        record(name, g, edges, "file", 0, R, seed, k)
    # reference-test style random instances (tests/test_baseline.py:22-38,
    # tests/test_acceptance.py:34-56 schemes and widths, padding 20 -> 24)
    cases = [
        ("er_const015_r32", 90, 6, "const:0.2", 1, 1, 32, 11, 6),
        ("er_const005_r64", 90, 6, "const:0.05", 2, 2, 64, 12, 4),
        ("er_uniform_r24", 90, 6, "uniform:0.1,0.7", 3, 3, 24, 13, 5),
        ("er_normal_r16", 90, 6, "normal:0.35,0.15", 4, 4, 16, 14, 5),
        ("er_wc_r40", 90, 6, "wc", 5, 5, 40, 15, 8),
        ("er_pad20", 60, 5, "const:0.2", 2, 0, 20, 1, 3),
        ("er_const1_r16", 80, 5, "const:1.0", 0, 0, 16, 0, 4),
        ("er_const0_r16", 80, 5, "const:0.0", 0, 0, 16, 0, 3),
        ("er_mid_300", 300, 6, "normal:0.25,0.15", 7, 8, 64, 3, 12),
        ("er_big_1000", 1000, 8, "uniform:0.02,0.5", 9, 10, 64, 5, 10),
        ("er_sub_2000", 2000, 6, "const:0.04", 11, 12, 128, 6, 15),
    ]
    for name, n, deg, scheme, gs, ws, R, seed, k in cases:
        g, edges = weighted_er(n, deg, scheme, gs, ws)
        record(name, g, edges, scheme, ws, R, seed, k)
    # benchmark configs C1 / C2 on this repo's Chung-Lu generator
    from paper_2008_03095_b200 import configs
    for cfg, full in (("c1", False), ("c2", False)):
        c = configs.CONFIGS[cfg]
        edges = configs.edges(cfg)
        g = apply_weights(Graph.from_edges(c.n, edges), parse_weight_scheme(c.weights),
                          rng_seed=c.seed)
        record(f"cfg_{cfg}", g, edges, c.weights, c.seed, c.R, 0, c.K, full=full)


if __name__ == "__main__":
    main()
