"""Golden fixtures for evaluate_seeds / sampling_cdf, made by running the
REFERENCE package (evaluation.py) in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_eval.py

Each evaluate case stores the graph (CSR + weights), the seeds, r_eval,
rng_seed, the reference's (mean, se) and its per-world reached counts (the
reference's own chunk workers run on its own spawned streams); each cdf case
stores the graph, X, the reference's SamplingCdf fields.  The config graphs
(c1, c2) are stored as their edge-list digest and rebuilt from this repo's
generator.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

import infmax.evaluation as ev  # noqa: E402
from infmax.graph import Graph, apply_weights, generate_er, parse_weight_scheme  # noqa: E402
from infmax.hashing import SimulationRandoms, build_hash_table  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_counts(g, seeds, r_eval, rng_seed):
    """The reference's per-world counts: its workers on its spawned streams
    (evaluation.py:117-133, n_threads=1)."""
    seeds = sorted({int(s) for s in seeds})
    cu, cv, probs = ev._canonical_probs(g)
    small = g.n <= ev._SMALL_N and len(probs) <= ev._SMALL_E
    worker = ev._closure_counts_small if small else ev._closure_counts_general
    starts = list(range(0, r_eval, ev._WORLD_CHUNK))
    streams = np.random.SeedSequence(rng_seed).spawn(len(starts))
    return np.concatenate([worker(g, seeds, probs, cu, cv, min(ev._WORLD_CHUNK, r_eval - s),
                                  np.random.default_rng(streams[i])) for i, s in enumerate(starts)])


def weighted_er(n, deg, scheme, graph_seed, weight_seed):
    return apply_weights(generate_er(n, deg, seed=graph_seed), parse_weight_scheme(scheme),
                         rng_seed=weight_seed)


def graph_arrays(g):
    return dict(n=np.int64(g.n), xadj=g.xadj, adj=g.adj, weights=g.weights)


def eval_case(name, g, seeds, r_eval, rng_seed, cfg=None):
    mean, se = ev.evaluate_seeds(g, seeds, r_eval, rng_seed=rng_seed)
    counts = ref_counts(g, seeds, r_eval, rng_seed)
    assert float(counts.mean()) == mean
    out = dict(seeds=np.asarray(seeds, np.int64), r_eval=np.int64(r_eval), rng_seed=np.int64(rng_seed),
               mean=np.float64(mean), se=np.float64(se), counts=counts.astype(np.int64))
    if cfg is None:
        out.update(graph_arrays(g))
    else:
        out.update(cfg=np.array(cfg), weights_sha=np.array(digest(g.weights)), adj_sha=np.array(digest(g.adj)))
    np.savez_compressed(HERE / f"eval_{name}.npz", **out)
    print(f"eval_{name}: n={g.n} m={g.m} r_eval={r_eval} mean={mean:.6f} se={se:.6f}")


def cdf_case(name, g, table, randoms, bins=100, cfg=None, broken=False):
    res = ev.sampling_cdf(g, table, randoms, bins=bins)
    out = dict(X=randoms.values, num_scored=np.int64(randoms.num_scored), bins=np.int64(bins),
               ks=np.float64(res.ks_distance), cdf=res.cdf, bin_uppers=res.bin_uppers,
               num_values=np.int64(res.num_values), broken=np.bool_(broken),
               R=np.int64(randoms.num_scored), master_seed=np.int64(randoms.master_seed))
    if cfg is None:
        out.update(graph_arrays(g))
    else:
        out.update(cfg=np.array(cfg), adj_sha=np.array(digest(g.adj)))
    np.savez_compressed(HERE / f"cdf_{name}.npz", **out)
    print(f"cdf_{name}: values={res.num_values} ks={res.ks_distance:.6g} ok={res.uniform_ok}")


def main():
    # evaluate_seeds: tiny-graph vectorised path, union-find path, multi-chunk
    g = weighted_er(40, 3, "uniform:0.2,0.8", 3, 1)
    eval_case("small40", g, [1, 7], 3000, 9)
    g = Graph.from_edges(5, [(0, 1), (1, 2), (3, 4)], 1.0)
    eval_case("kat_w1", g, [0, 3], 100, 0)
    g = Graph.from_edges(3, [(0, 1), (1, 2)], [0.5, 0.25])
    eval_case("kat_half", g, [1], 5000, 2)
    g = weighted_er(200, 6, "const:0.1", 1, 0)
    eval_case("er200", g, [0, 5, 9], 10_000, 3)
    g = weighted_er(300, 6, "normal:0.25,0.15", 7, 8)
    eval_case("er300_dup", g, [12, 4, 4, 280, 12], 4200, 11)
    g = weighted_er(1000, 8, "uniform:0.02,0.5", 9, 10)
    eval_case("er1000", g, [3, 17, 400, 999], 8200, 5)
    from paper_2008_03095_b200 import configs
    c = configs.CONFIGS["c1"]
    g = apply_weights(Graph.from_edges(c.n, configs.edges("c1")), parse_weight_scheme(c.weights),
                      rng_seed=c.seed)
    seeds = np.load(HERE / "cfg_c1.npz")["seeds"].tolist()
    eval_case("cfg_c1", g, seeds, 4500, 1, cfg="c1")
    # sampling_cdf: reference-test shapes, a degenerate table, a strided config
    g = generate_er(2000, 10, seed=4)
    cdf_case("er2000", g, build_hash_table(g), SimulationRandoms(256, master_seed=0))
    broken = build_hash_table(g)
    broken.hashes[:] = 0
    cdf_case("er2000_broken", g, broken, SimulationRandoms(256, master_seed=0), broken=True)
    g = generate_er(100, 4, seed=1)
    cdf_case("er100_b50", g, build_hash_table(g), SimulationRandoms(8, master_seed=2), bins=50)
    c = configs.CONFIGS["c2"]
    g = Graph.from_edges(c.n, configs.edges("c2"))
    cdf_case("cfg_c2", g, build_hash_table(g), SimulationRandoms(c.R, master_seed=0), cfg="c2")


if __name__ == "__main__":
    main()
