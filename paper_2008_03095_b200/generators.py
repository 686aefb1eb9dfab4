"""Seeded synthetic graphs for the benchmark configurations (BASELINE.json).

The reference ships Erdos-Renyi and R-MAT generators (graph.py:444-491) but
no Chung-Lu; the paper's datasets are not available here, so every config is
a seeded synthetic stand-in with the published shape.  All
generators return a list of distinct undirected edges without self-loops,
from which ``Graph.from_edges`` (device CSR builder) builds the graph.
"""

from __future__ import annotations

import numpy as np

__all__ = ["chung_lu_edges", "rmat_edges", "er_edges", "unique_first"]


def unique_first(u: np.ndarray, v: np.ndarray, n: int) -> np.ndarray:
    """Indices of the first draw of every unordered pair, in draw order."""
    key = np.minimum(u, v).astype(np.int64) * np.int64(n) + np.maximum(u, v)
    _, first = np.unique(key, return_index=True)
    first.sort()
    return first


def _accumulate(draw, n: int, target: int, batch: int):
    """Draw (u, v) batches until ``target`` distinct non-loop pairs exist."""
    us, vs = np.empty(0, np.int64), np.empty(0, np.int64)
    while len(us) < target:
        u, v = draw(max(batch, int(1.25 * (target - len(us)))))
        keep = u != v
        us = np.concatenate([us, u[keep]])
        vs = np.concatenate([vs, v[keep]])
        first = unique_first(us, vs, n)
        us, vs = us[first], vs[first]
    return np.column_stack([us[:target], vs[:target]])


def chung_lu_edges(n: int, m: int, gamma: float, seed: int) -> np.ndarray:
    """Chung-Lu power-law graph: expected degree of vertex i proportional to
    (i + 1) ** (-1 / (gamma - 1)) (hubs get low ids); endpoints drawn
    independently proportional to that weight, self-loops and repeats
    dropped, first ``m`` distinct edges kept."""
    rng = np.random.default_rng(seed)
    w = (np.arange(1, n + 1, dtype=np.float64)) ** (-1.0 / (gamma - 1.0))
    cdf = np.cumsum(w)
    cdf /= cdf[-1]

    def draw(k):
        u = np.searchsorted(cdf, rng.random(k), side="right")
        v = np.searchsorted(cdf, rng.random(k), side="right")
        return np.minimum(u, n - 1).astype(np.int64), np.minimum(v, n - 1).astype(np.int64)

    return _accumulate(draw, n, m, 1 << 16)


def _rmat_draw(rng, scale: int, k: int, probs):
    a, b, c, _ = probs
    total = sum(probs)
    ca, cb, cc = a / total, (a + b) / total, (a + b + c) / total
    u = np.zeros(k, np.int64)
    v = np.zeros(k, np.int64)
    for _level in range(scale):
        x = rng.random(k, dtype=np.float32)
        right = ((x >= ca) & (x < cb)) | (x >= cc)      # quadrants b, d
        down = x >= cb                                   # quadrants c, d
        u = (u << 1) | down
        v = (v << 1) | right
    return u, v


def rmat_edges(scale: int, seed: int, probs=(0.57, 0.19, 0.19, 0.05), *,
               m: int | None = None, edge_factor: int | None = None,
               chunk: int = 1 << 22) -> np.ndarray:
    """Symmetrised, deduplicated R-MAT graph on 2**scale vertices.

    ``m`` -> draw until exactly m distinct undirected edges (first draws kept);
    ``edge_factor`` -> draw edge_factor * 2**scale pairs once and keep every
    distinct non-loop pair (Graph500 style)."""
    n = 1 << scale
    rng = np.random.default_rng(seed)
    if m is not None:
        return _accumulate(lambda k: _rmat_draw(rng, scale, k, probs), n, m, 1 << 16)
    if edge_factor is None:
        raise ValueError("need m or edge_factor")
    total = edge_factor * n
    keys = []
    for start in range(0, total, chunk):
        u, v = _rmat_draw(rng, scale, min(chunk, total - start), probs)
        keep = u != v
        lo = np.minimum(u[keep], v[keep])
        hi = np.maximum(u[keep], v[keep])
        keys.append(np.unique((lo << scale) | hi))
    key = np.unique(np.concatenate(keys))
    return np.column_stack([key >> scale, key & ((1 << scale) - 1)])


def er_edges(n: int, m: int, seed: int) -> np.ndarray:
    """Erdos-Renyi G(n, m): uniform pairs, first m distinct non-loop pairs."""
    rng = np.random.default_rng(seed)
    return _accumulate(lambda k: (rng.integers(0, n, k), rng.integers(0, n, k)), n, m, 1 << 16)
