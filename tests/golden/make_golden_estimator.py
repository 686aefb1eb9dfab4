"""Golden fixtures for the estimator / validation layer, made by running the
REFERENCE package (estimator.py, validation.py) in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_estimator.py
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from infmax.estimator import InfluenceMaximizer
from infmax.validation import as_graph

HERE = Path(__file__).resolve().parent


def main():
    rng = np.random.default_rng(11)
    ids = rng.integers(-500, 500, size=300)
    rows = []
    for _ in range(1500):
        a, b = rng.choice(ids, size=2)
        rows.append((a, b, round(float(rng.random()), 4)))
    rows += [(ids[3], ids[3], 0.5), tuple(rows[10])]          # a self-loop and a duplicate
    arr = np.array(rows, dtype=np.float64)
    g = as_graph(arr)
    g2 = as_graph(arr[:, :2].astype(np.int64))
    cases = {}
    for name, (scheme, k, r, seed, X) in {
        "const": ("const:0.3", 4, 64, 2, arr[:, :2].astype(np.int64)),
        "file": ("file", 3, 40, 5, arr),
        "wc": ("wc", 5, 128, 0, arr[:, :2].astype(np.int64)),
    }.items():
        m = InfluenceMaximizer(k=k, num_simulations=r, weight_scheme=scheme, random_state=seed).fit(X)
        cases[name] = dict(seeds=m.seeds_, idx=m.seed_indices_, spread=np.float64(m.expected_spread_),
                           se=np.float64(m.expected_spread_se_), score=np.float64(m.score(r_eval=3000)),
                           k=np.int64(k), r=np.int64(r), seed=np.int64(seed), scheme=np.array(scheme))
    out = dict(arr=arr, xadj=g.xadj, adj=g.adj, weights=g.weights, orig=g.orig_ids,
               xadj2=g2.xadj, adj2=g2.adj, weights2=g2.weights, orig2=g2.orig_ids)
    for name, c in cases.items():
        for key, v in c.items():
            out[f"{name}_{key}"] = v
    np.savez_compressed(HERE / "est_cases.npz", **out)
    print({n: (c["seeds"].tolist(), float(c["spread"]), float(c["score"])) for n, c in cases.items()})


if __name__ == "__main__":
    main()
