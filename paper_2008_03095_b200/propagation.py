"""Fused sample + connected-components over R implicit samples (K3) and the
memoized component-size gains (K4/K5), behind the reference's entry points
(reference propagation.py:260-403).

``propagate`` returns the same (n, width) int32 label matrix as the
reference -- in every lane the minimum vertex id of the vertex's component
in the sample ``(X[r] ^ hash) < thr`` -- but computes it on the GPU with a
single fused union-find pass over all lanes (see csrc/cc.cu), so its
``PropagateStats`` report one label-moving sweep ("hook") plus the
no-change sweep that proves convergence ("verify"), instead of the
reference's index/dense/sparse sweep mix.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .context import DeviceContext, empty_graph
from .graph import Graph
from .hashing import LANE_WIDTH, EdgeHashTable, SimulationRandoms

__all__ = ["PropagateStats", "propagate", "component_sizes", "initial_marginal_gains",
           "component_sizes_and_gains", "lane_label_step", "dump_labels", "load_labels"]


@dataclass
class PropagateStats:
    """Sweep count, per-sweep changed (vertex, lane) pairs, modes, label sums
    (reference propagation.py:49-56)."""

    sweeps: int = 0
    changed_pairs: list = field(default_factory=list)
    modes: list = field(default_factory=list)
    label_sums: list = field(default_factory=list)


def _width(randoms, num_simulations) -> int:
    """Validated propagation width (reference propagation.py:267-273)."""
    num_lanes = randoms.padded if num_simulations is None else int(num_simulations)
    if num_lanes < 1 or num_lanes % LANE_WIDTH:
        raise ValueError(f"simulation width {num_lanes} not a multiple of {LANE_WIDTH}")
    if num_lanes > randoms.padded:
        raise ValueError(f"simulation width {num_lanes} exceeds {randoms.padded} randoms")
    return num_lanes


def propagated_context(g: Graph, table: EdgeHashTable | None, X: np.ndarray, num_scored: int,
                       verify: bool = False, stats: bool = False, lane0: int = 0,
                       fuse_memo: bool = False, defer_spec: bool = False):
    """Create a context for lanes X on g, bind the hash table, propagate
    (with the memo fused into a tiled compression when ``fuse_memo``)."""
    if table is not None:
        table.bind(g)
    ctx = DeviceContext(g, X, num_scored, lane0)
    if fuse_memo:
        ctx.set_fuse_memo(True)
    if defer_spec:          # the caller checks ctx.spec_settle() before trusting results
        ctx.spec_defer(True)
    st = ctx.propagate(verify=verify, stats=stats)
    return ctx, st


def propagate(g: Graph, table: EdgeHashTable, randoms: SimulationRandoms,
              num_simulations: int | None = None, n_threads: int = 1,
              return_stats: bool = False):
    """Converged (n, width) int32 min-id label matrix (reference
    propagation.py:260-321).  ``n_threads`` is accepted for signature
    compatibility; the device decides its own parallelism."""
    num_lanes = _width(randoms, num_simulations)
    stats = PropagateStats()
    if g.m == 0:
        labels = np.repeat(np.arange(g.n, dtype=np.int32)[:, None], num_lanes, axis=1)
        return (labels, stats) if return_stats else labels
    X = np.ascontiguousarray(randoms.values[:num_lanes])
    ctx, st = propagated_context(g, table, X, num_lanes, verify=return_stats, stats=return_stats)
    labels = ctx.labels()
    ctx.close()
    if return_stats:
        stats.sweeps, stats.changed_pairs, stats.label_sums, stats.modes = st
        return labels, stats
    return labels


def _host_label_context(labels: np.ndarray, num_scored: int, sizes=None) -> DeviceContext:
    labels = np.ascontiguousarray(labels, dtype=np.int32)
    if labels.ndim != 2:
        raise ValueError("labels must be an (n, R) matrix")
    n, width = labels.shape
    if width < 1:
        raise ValueError("labels need at least one lane")
    ctx = DeviceContext(empty_graph(n), np.zeros(width, np.int32), num_scored)
    ctx.load_labels(labels, sizes)
    return ctx


def component_sizes(labels: np.ndarray) -> np.ndarray:
    """sizes[l, r] = number of vertices labelled l in lane r, shape (n, R)
    (reference propagation.py:349-356); device histogram."""
    ctx = _host_label_context(labels, labels.shape[1])
    out = ctx.sizes()
    ctx.close()
    return out


def initial_marginal_gains(labels: np.ndarray, sizes: np.ndarray,
                           num_scored: int | None = None) -> np.ndarray:
    """gains[v] = sum over scored lanes of sizes[labels[v, r], r], int64
    (reference propagation.py:359-368); device gather-reduce."""
    num_scored = labels.shape[1] if num_scored is None else int(num_scored)
    ctx = _host_label_context(labels, num_scored, sizes)
    gains = ctx.memoize()
    ctx.close()
    return gains


def component_sizes_and_gains(labels: np.ndarray, num_scored: int | None = None):
    """(sizes (n, R) int32, gains int64[n]) in one device pass over the
    labels (reference propagation.py:371-390)."""
    num_scored = labels.shape[1] if num_scored is None else int(num_scored)
    ctx = _host_label_context(labels, num_scored)
    gains = ctx.memoize()
    sizes = ctx.sizes()
    ctx.close()
    return sizes, gains


def lane_label_step(g: Graph, u: int, v: int, r0: int, labels: np.ndarray,
                    table: EdgeHashTable, randoms: SimulationRandoms,
                    thresholds: np.ndarray | None = None) -> bool:
    """One push of edge (u, v) into v for the LANE_WIDTH simulations at r0
    (Alg. 5 semantics, reference propagation.py:324-346).  A single-edge,
    8-lane illustration of the sampler predicate; not used by ``propagate``."""
    if r0 % LANE_WIDTH or r0 + LANE_WIDTH > labels.shape[1]:
        raise ValueError(f"batch start {r0} invalid for width {labels.shape[1]}")
    slot = g.slot(u, v)
    if thresholds is None:
        from .hashing import slot_thresholds
        thresholds = slot_thresholds(g)
    lanes = slice(r0, r0 + LANE_WIDTH)
    live = (randoms.values[lanes] ^ np.int32(table.hashes[slot])) < thresholds[slot]
    lu, lv = labels[u, lanes], labels[v, lanes]
    new = np.where(live & (lu < lv), lu, lv)
    changed = bool((new != lv).any())
    labels[v, lanes] = new
    return changed


def dump_labels(labels: np.ndarray, path) -> None:
    """Binary dump: little-endian u64 n, R, then row-major int32 labels
    (reference propagation.py:393-397)."""
    arr = np.ascontiguousarray(labels, dtype="<i4")
    with open(path, "wb") as fh:
        fh.write(np.asarray(arr.shape, dtype="<u8").tobytes())
        fh.write(arr.tobytes())


def load_labels(path) -> np.ndarray:
    raw = np.fromfile(path, dtype=np.uint8)
    n, r = (int(x) for x in raw[:16].view("<u8"))
    return raw[16:].view("<i4").reshape(n, r).astype(np.int32)
