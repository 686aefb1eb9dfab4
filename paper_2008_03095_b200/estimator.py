"""Scikit-learn-style estimator and input validation over the device path
(reference estimator.py:1-106, validation.py:1-85).

``InfluenceMaximizer.fit`` runs ``run_fused`` (device propagate + memo + CELF)
and ``score`` runs ``evaluate_seeds`` on fresh worlds on the device; the
inputs (a Graph, a graph file, or an edge array) are coerced exactly as the
reference coerces them.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
from sklearn.base import BaseEstimator

from ._lib import ConstraintError
from .evaluation import evaluate_seeds
from .graph import Graph
from .io import load_graph
from .pipeline import run_fused
from .weights import FromFile, apply_weights, parse_weight_scheme

__all__ = ["InfluenceMaximizer", "as_graph", "check_graph", "check_num_seeds", "check_simulations"]


def as_graph(X) -> Graph:
    """A Graph, a path to an edge list / CSR cache, or a non-empty (k, 2|3)
    edge array (ids compacted by first appearance, self-loops dropped,
    duplicates collapse to the first occurrence) (validation.py:12-46)."""
    if isinstance(X, Graph):
        return X
    if isinstance(X, (str, Path)):
        return load_graph(X)
    arr = np.asarray(X)
    if arr.ndim != 2 or arr.shape[1] not in (2, 3) or arr.shape[0] == 0:
        raise ValueError("X must be a Graph, a graph file path, or a non-empty (k, 2|3) edge array")
    ab = np.array([[int(r[0]), int(r[1])] for r in arr], dtype=np.int64) if arr.dtype == object \
        else arr[:, :2].astype(np.int64)
    keep = ab[:, 0] != ab[:, 1]
    rows = np.flatnonzero(keep)
    if len(rows) == 0:
        raise ValueError("edge array contains no usable edges")
    seq = ab[rows].ravel()                          # endpoints in order of appearance
    uniq, first = np.unique(seq, return_index=True)
    order = np.argsort(first, kind="stable")
    orig = uniq[order]
    compact = np.empty(len(uniq), np.int64)
    compact[order] = np.arange(len(uniq))
    cu = compact[np.searchsorted(uniq, ab[rows, 0])]
    cv = compact[np.searchsorted(uniq, ab[rows, 1])]
    key = np.minimum(cu, cv) * len(uniq) + np.maximum(cu, cv)
    _, firstk = np.unique(key, return_index=True)
    sel = np.sort(firstk)
    ws = arr[rows[sel], 2].astype(np.float64) if arr.shape[1] == 3 else np.ones(len(sel))
    return Graph.from_edges(len(uniq), np.column_stack([cu[sel], cv[sel]]), ws, orig)


def check_graph(g: Graph) -> Graph:
    """Offsets, symmetry and weight range (validation.py:49-56)."""
    if g.xadj[0] != 0 or g.xadj[-1] != g.m or (np.diff(g.xadj) < 0).any():
        raise ValueError("corrupt CSR offsets")
    g.reciprocal_slots  # raises GraphFormatError if not symmetric
    if g.m and (g.weights.min() < 0.0 or g.weights.max() > 1.0):
        raise ConstraintError("weights must lie in [0, 1]")
    return g


def check_num_seeds(k: int, n: int) -> int:
    k = int(k)
    if k < 1:
        raise ConstraintError(f"need at least one seed, got k={k}")
    if k > n:
        raise ConstraintError(f"k={k} exceeds vertex count n={n}")
    return k


def check_simulations(r: int) -> int:
    r = int(r)
    if r < 1:
        raise ConstraintError(f"simulation count must be positive, got {r}")
    return r


class InfluenceMaximizer(BaseEstimator):
    """Greedy influence maximization under the independent cascade model
    (reference estimator.py:14-106); parameters and fitted attributes as
    there: ``seeds_``, ``seed_indices_``, ``expected_spread_``,
    ``expected_spread_se_``, ``n_vertices_``, ``trace_``, ``graph_``."""

    def __init__(self, k: int = 10, num_simulations: int = 256, weight_scheme: str = "wc",
                 random_state: int = 0, n_threads: int = 1):
        self.k = k
        self.num_simulations = num_simulations
        self.weight_scheme = weight_scheme
        self.random_state = random_state
        self.n_threads = n_threads

    def fit(self, X, y=None):
        """Select seeds on a graph given as a Graph, file path, or edge array."""
        g = check_graph(as_graph(X))
        k = check_num_seeds(self.k, g.n)
        r = check_simulations(self.num_simulations)
        scheme = parse_weight_scheme(self.weight_scheme)
        if not isinstance(scheme, FromFile):
            g = apply_weights(g, scheme, rng_seed=self.random_state)
        run = run_fused(g, k, num_simulations=r, master_seed=self.random_state, n_threads=int(self.n_threads))
        self.graph_ = g
        self.n_vertices_ = g.n
        self.seed_indices_ = np.asarray(run.seeds, dtype=np.int64)
        self.seeds_ = np.asarray(run.original_seed_ids(), dtype=np.int64)
        self.expected_spread_ = run.spread
        self.expected_spread_se_ = run.spread_se
        self.trace_ = run.selection.trace
        return self

    def predict(self, X=None):
        """Fitted seeds (original ids); X is accepted for pipeline parity."""
        self._check_fitted()
        return self.seeds_

    def score(self, X=None, y=None, r_eval: int = 10_000, random_state: int | None = None) -> float:
        """Independent Monte-Carlo estimate of the fitted seeds' spread on
        fresh worlds (evaluate_seeds on the device)."""
        self._check_fitted()
        seed = self.random_state + 1 if random_state is None else random_state
        mean, _ = evaluate_seeds(self.graph_, self.seed_indices_.tolist(), r_eval, seed,
                                 n_threads=int(self.n_threads))
        return mean

    def _check_fitted(self):
        if not hasattr(self, "seeds_"):
            raise AttributeError("estimator is not fitted; call fit first")
