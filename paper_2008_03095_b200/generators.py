"""Seeded synthetic graphs for the benchmark configurations (BASELINE.json).

The reference ships Erdos-Renyi and R-MAT generators (graph.py:444-491) but
no Chung-Lu, and the paper's datasets are not available here, so every
config is a seeded synthetic stand-in with the published shape.

Random numbers are counter-based SplitMix64 values ``rnd(seed, index)``: a
candidate depends only on its index, so the device generator (csrc/gen.cu,
``device_graph``) and the numpy restatement below (``edges``, used by the CPU
reference arm and the tests) produce the same edges bit for bit:

* Erdos-Renyi: u = hi64(rnd(s, 2i) * n), v = hi64(rnd(s, 2i+1) * n)
* R-MAT: level l of candidate i draws unit(rnd(s, 64 i + l)) and picks the
  quadrant a | b | c | d from the cumulative probabilities
* Chung-Lu: u = #{cdf <= unit(rnd(s, 2i))} (searchsorted right), v likewise
  with 2i+1; cdf = normalised cumulative expected degrees (i+1)^(-1/(g-1))

Self-loops are dropped and unordered pairs deduplicated keeping the first
draw.  ``m > 0``: the first m distinct pairs in draw order; ``m == 0``: every
distinct pair among ``draws`` candidates (Graph500 style).
"""

from __future__ import annotations

import ctypes

import numpy as np

__all__ = ["ER", "RMAT", "CHUNG_LU", "edges", "device_graph", "chung_lu_cdf", "er_edges"]

ER, RMAT, CHUNG_LU = 0, 1, 2
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix64(z):
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _rnd(seed: int, idx: np.ndarray) -> np.ndarray:
    return _mix64(_mix64(np.uint64(seed)) ^ idx.astype(np.uint64))


def _unit(r: np.ndarray) -> np.ndarray:
    return (r >> np.uint64(11)).astype(np.float64) * 2.0**-53


def _below(r: np.ndarray, n: int) -> np.ndarray:
    nn = np.uint64(n)
    with np.errstate(over="ignore"):
        return ((r >> np.uint64(32)) * nn + (((r & np.uint64(0xFFFFFFFF)) * nn) >> np.uint64(32))) >> np.uint64(32)


def chung_lu_cdf(n: int, gamma: float) -> np.ndarray:
    w = np.arange(1, n + 1, dtype=np.float64) ** (-1.0 / (gamma - 1.0))
    cdf = np.cumsum(w)
    return cdf / cdf[-1]


def _rmat_cuts(probs):
    a, b, c, d = (float(x) for x in probs)
    tot = a + b + c + d
    return a / tot, (a + b) / tot, (a + b + c) / tot


def _candidates(kind, n, seed, first, count, probs=None, cdf=None):
    i = np.arange(first, first + count, dtype=np.uint64)
    if kind == ER:
        u = _below(_rnd(seed, 2 * i), n)
        v = _below(_rnd(seed, 2 * i + np.uint64(1)), n)
    elif kind == RMAT:
        scale = int(n).bit_length() - 1
        ca, cb, cc = _rmat_cuts(probs)
        u = np.zeros(count, np.uint64)
        v = np.zeros(count, np.uint64)
        for level in range(scale):
            x = _unit(_rnd(seed, np.uint64(64) * i + np.uint64(level)))
            down = x >= cb
            right = ((x >= ca) & (x < cb)) | (x >= cc)
            u = (u << np.uint64(1)) | down.astype(np.uint64)
            v = (v << np.uint64(1)) | right.astype(np.uint64)
    else:
        x1 = _unit(_rnd(seed, 2 * i))
        x2 = _unit(_rnd(seed, 2 * i + np.uint64(1)))
        u = np.minimum(np.searchsorted(cdf, x1, side="right"), n - 1).astype(np.uint64)
        v = np.minimum(np.searchsorted(cdf, x2, side="right"), n - 1).astype(np.uint64)
    lo, hi = np.minimum(u, v), np.maximum(u, v)
    key = lo * np.uint64(n) + hi
    key[u == v] = _M64
    return key


def edges(kind: int, n: int, m: int, seed: int, draws: int = 0, probs=None, cdf=None,
          chunk: int = 1 << 23) -> np.ndarray:
    """(k, 2) int64 distinct undirected edges, the same as the device generator."""
    if m > 0 and draws <= 0:
        draws = m + m // 4 + 4096
    while True:
        keys = np.concatenate([_candidates(kind, n, seed, s, min(chunk, draws - s), probs, cdf)
                               for s in range(0, draws, chunk)])
        # first draw of every distinct key (np.unique(return_index) without
        # its slow generic path on tens of millions of uint64 keys)
        order = np.argsort(keys, kind="stable")
        srt = keys[order]
        head = np.ones(len(srt), bool)
        head[1:] = srt[1:] != srt[:-1]
        head &= srt != _M64
        uniq, first = srt[head], order[head]
        if m == 0 or len(uniq) >= m:
            break
        draws = min(draws + draws // 2, 1 << 31)
    if m > 0:
        order = np.argsort(first, kind="stable")[:m]
        uniq = uniq[order]
    return np.column_stack([(uniq // np.uint64(n)).astype(np.int64), (uniq % np.uint64(n)).astype(np.int64)])


def device_graph(kind: int, n: int, m: int, seed: int, draws: int = 0, probs=None, cdf=None):
    """Generate on the device and build the CSR there (unit weights)."""
    from . import _lib
    from ._lib import check, ptr
    from .graph import DeviceGraph, Graph
    _lib.require_device()
    dev = _lib.current_device()
    par = None if probs is None else np.ascontiguousarray(probs, dtype=np.float64)
    cdfa = None if cdf is None else np.ascontiguousarray(cdf, dtype=np.float64)
    h = ctypes.c_void_p()
    check(_lib.load().imx_graph_generate(dev, kind, int(n), int(m), int(draws), int(seed) & (2**64 - 1),
                                         ptr(par), ptr(cdfa), ctypes.byref(h)))
    dg = DeviceGraph(h, dev)
    nn, m2 = dg.dims()
    xadj = np.empty(nn + 1, np.int64)
    adj = np.empty(m2, np.int32)
    w = np.empty(m2, np.float64)
    check(_lib.load().imx_graph_get_csr(h, ptr(xadj), ptr(adj), ptr(w)))
    return Graph(xadj, adj, w, np.arange(nn, dtype=np.int64), dg)


def er_edges(n: int, m: int, seed: int) -> np.ndarray:
    """Erdos-Renyi G(n, m) edge list (counter-based streams)."""
    return edges(ER, n, m, seed)
