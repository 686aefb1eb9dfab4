"""Greedy CELF seed selection over memoized component labels, on the device
(reference selection.py:1-159).

``select_seeds`` runs the round-based exact CELF of csrc/cc.cu
(imx_celf_select): per round it evaluates the top-priority vertex and then
every vertex whose stale priority could still beat that fresh gain, commits
the lexicographic argmax (max gain, then min id), and rebuilds the lazy
heap's dequeue trace exactly.  Gains are integer sums in
vertex x simulation units, as in the reference.

``SeedState`` / ``marginal_gain`` / ``commit_seed`` keep the reference's
per-vertex API; the state is a device context holding the covered-component
bitmaps, attached on first use.
"""

from __future__ import annotations

import csv
import heapq
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np

from ._lib import ConstraintError
from .context import DeviceContext, empty_graph

__all__ = ["TraceRecord", "SeedState", "marginal_gain", "commit_seed", "recompute_sigma",
           "SelectionResult", "select_seeds", "write_trace_csv"]


@dataclass
class TraceRecord:
    """One CELF dequeue (reference selection.py:25-33)."""

    vertex: int
    stale_gain: int
    fresh_gain: int
    committed: bool
    seeds_before: int


class SeedState:
    """Seeds, running sigma and per-lane owned labels (reference
    selection.py:36-60).  ``owned[l, r]`` is materialised from the device
    bitmap when read."""

    def __init__(self, num_scored: int, owned=None, seeds=None, sigma: int = 0,
                 *, n: int | None = None, ctx: DeviceContext | None = None, per_sim=None):
        self.num_scored = int(num_scored)
        self._owned = owned
        self._n = n if n is not None else (None if owned is None else owned.shape[0])
        self.seeds = list(seeds) if seeds is not None else []
        self.sigma = int(sigma)
        self._ctx = ctx
        self._ctx_key = None
        self._per_sim = per_sim
        self._shard = None        # (ctx, comm): this rank's lane window of a sharded run

    @classmethod
    def empty(cls, n: int, num_scored: int) -> "SeedState":
        return cls(num_scored, n=n)

    @property
    def owned(self) -> np.ndarray:
        if self._shard is not None:
            from .celf import gather_owned
            return gather_owned(*self._shard)
        if self._ctx is not None:
            return self._ctx.owned()
        if self._owned is None:
            self._owned = np.zeros((self._n, self.num_scored), dtype=bool)
        return self._owned

    @owned.setter
    def owned(self, value):
        self._owned = np.asarray(value, dtype=bool)
        self._ctx = None
        self._shard = None

    def seed_label_sets(self) -> list:
        """Per-simulation sets of owned labels."""
        out = [set() for _ in range(self.num_scored)]
        labels, lanes = np.nonzero(self.owned)
        for l, r in zip(labels.tolist(), lanes.tolist()):
            out[r].add(l)
        return out

    # -- device attachment for the per-vertex API ---------------------------------
    def _attach(self, labels: np.ndarray, sizes: np.ndarray | None) -> DeviceContext:
        key = (id(labels), None if sizes is None else id(sizes))
        if self._ctx is not None and (self._ctx_key == key or (sizes is None and self._ctx_key and self._ctx_key[0] == key[0])):
            return self._ctx
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        n, width = labels.shape
        if self.num_scored > width:
            raise ValueError(f"num_scored {self.num_scored} exceeds label width {width}")
        owned_before = None if self._ctx is None else self._ctx.owned()
        if owned_before is None and self._owned is not None:
            owned_before = self._owned
        ctx = DeviceContext(empty_graph(n), np.zeros(width, np.int32), self.num_scored)
        ctx.load_labels(labels, sizes)
        ctx.celf_reset(np.zeros(n, np.int64))
        for s in self.seeds:
            ctx.commit(s)
        if owned_before is not None and owned_before.any():
            # reproduce ownership that was set outside commit_seed
            mine = ctx.owned()
            if not np.array_equal(mine, owned_before):
                raise ValueError("state.owned is not reproducible from state.seeds")
        self._ctx, self._ctx_key = ctx, key
        return ctx

    @property
    def per_sim(self) -> np.ndarray:
        if self._ctx is not None:
            return self._ctx.per_sim()
        return self._per_sim


def marginal_gain(u: int, labels: np.ndarray, sizes: np.ndarray, state: SeedState) -> int:
    """Spread gained by adding u: its component size in every scored lane
    whose component is not owned yet (reference selection.py:63-70)."""
    ctx = state._attach(labels, sizes)
    return int(ctx.eval_gains(np.array([u], np.int32))[0])


def commit_seed(u: int, gain: int, labels: np.ndarray, state: SeedState) -> SeedState:
    """Own u's component in every scored lane and bank ``gain``
    (reference selection.py:73-81)."""
    if u in state.seeds:
        raise AssertionError(f"vertex {u} committed twice")
    ctx = state._attach(labels, None)
    ctx.commit(int(u))
    state.seeds.append(int(u))
    state.sigma += int(gain)
    return state


def recompute_sigma(labels: np.ndarray, state: SeedState) -> int:
    """Independent recount of vertices in owned components (reference
    selection.py:84-88): gathers ``owned`` through the label matrix."""
    cols = np.arange(state.num_scored)
    return int(state.owned[labels[:, : state.num_scored], cols].sum(dtype=np.int64))


@dataclass
class SelectionResult:
    seeds: list
    sigma: int
    num_scored: int
    trace: list
    gains: list
    state: SeedState

    @property
    def spread(self) -> float:
        """sigma / R in vertices (reference selection.py:100-103)."""
        return self.sigma / self.num_scored

    def spread_se(self, labels=None, sizes=None) -> float:
        """Standard error over the scored simulations of the per-lane covered
        totals (reference selection.py:105-112); per_sim comes from the
        device (K8)."""
        per_sim = self.state.per_sim
        if per_sim is None:
            cols = np.arange(self.num_scored)
            per_sim = self.state.owned[labels[:, : self.num_scored], cols].sum(axis=0, dtype=np.int64)
        if self.num_scored < 2:
            return 0.0
        per_sim = np.asarray(per_sim, dtype=np.int64)
        return float(per_sim.std(ddof=1) / np.sqrt(self.num_scored))


def _check_k(k: int, n: int) -> int:
    if k < 1:
        raise ConstraintError(f"need at least one seed, got k={k}")
    if k > n:
        raise ConstraintError(f"k={k} exceeds vertex count n={n}")
    return int(k)


class TraceList(Sequence):
    """The CELF dequeue trace as a read-only list of TraceRecord, built from
    the (T, 5) int64 array the device returns; records are created on
    access, so a caller that never reads the trace never pays for it."""

    def __init__(self, arr: np.ndarray):
        self.array = np.asarray(arr, dtype=np.int64).reshape(-1, 5)
        self._cache = None

    def _records(self) -> list:
        if self._cache is None:
            self._cache = [TraceRecord(v, s, f, bool(c), t) for v, s, f, c, t in self.array.tolist()]
        return self._cache

    def __len__(self) -> int:
        return len(self.array)

    def __getitem__(self, i):
        return self._records()[i]

    def __iter__(self):
        return iter(self._records())

    def __eq__(self, other):
        return list(self) == list(other)

    def __repr__(self):
        return f"TraceList({len(self)} records)"


def trace_records(trace: np.ndarray) -> TraceList:
    return TraceList(trace)


def result_from_context(ctx: DeviceContext, seeds, gains, trace, num_scored: int) -> SelectionResult:
    state = SeedState(num_scored, n=ctx.n, seeds=[int(s) for s in seeds],
                      sigma=int(np.sum(gains, dtype=np.int64)), ctx=ctx)
    return SelectionResult(list(state.seeds), state.sigma, num_scored, trace_records(trace),
                           [int(x) for x in gains], state)


def select_seeds(g, labels: np.ndarray, sizes: np.ndarray, initial_gains: np.ndarray, k: int,
                 num_scored: int | None = None) -> SelectionResult:
    """Pick k seeds greedily; ties break toward the smaller vertex id
    (reference selection.py:115-149).  Runs on the device over the given
    label/size matrices."""
    n = g.n
    _check_k(k, n)
    labels = np.asarray(labels)
    num_scored = labels.shape[1] if num_scored is None else int(num_scored)
    ctx = DeviceContext(empty_graph(n), np.zeros(labels.shape[1], np.int32), num_scored)
    ctx.load_labels(labels, sizes)
    init = np.asarray(initial_gains, dtype=np.int64)
    if init.shape != (n,):
        raise ValueError(f"initial_gains shape {init.shape} != ({n},)")
    memo = ctx.memoize(want_gains=True)
    if (init < memo).any():
        # priorities that under-estimate some gain: the round-based CELF
        # needs upper bounds, so run the reference's lazy heap itself, every
        # marginal gain and commit still on the device
        seeds, gains, trace = _lazy_heap(ctx, init, k)
    else:
        ctx.celf_reset(init)
        seeds, gains, trace = ctx.celf_select(k)
    return result_from_context(ctx, seeds, gains, trace, num_scored)


def _lazy_heap(ctx: DeviceContext, initial_gains: np.ndarray, k: int):
    """select_seeds' heap loop (reference selection.py:128-147) with
    marginal_gain / commit_seed on the device: exact for any priorities."""
    ctx.celf_reset(None)
    queue = [(-int(g), v) for v, g in enumerate(initial_gains.tolist())]
    heapq.heapify(queue)
    fresh_at = np.zeros(len(initial_gains), dtype=np.int64)
    seeds, gains, trace = [], [], []
    while len(seeds) < k:
        neg, u = heapq.heappop(queue)
        stale = -neg
        if fresh_at[u] == len(seeds):
            ctx.commit(u)
            trace.append((u, stale, stale, 1, len(seeds)))
            seeds.append(u)
            gains.append(stale)
        else:
            fresh = int(ctx.eval_gains(np.array([u], np.int32))[0])
            fresh_at[u] = len(seeds)
            heapq.heappush(queue, (-fresh, u))
            trace.append((u, stale, fresh, 0, len(seeds)))
    return (np.asarray(seeds, np.int32), np.asarray(gains, np.int64),
            np.asarray(trace, np.int64).reshape(-1, 5))


def write_trace_csv(trace: list, path) -> None:
    """vertex, stale_gain, fresh_gain, committed, seeds_before per dequeue."""
    with open(path, "w", newline="", encoding="utf-8") as fh:
        out = csv.writer(fh)
        out.writerow(["vertex", "stale_gain", "fresh_gain", "committed", "seeds_before"])
        out.writerows([t.vertex, t.stale_gain, t.fresh_gain, int(t.committed), t.seeds_before]
                      for t in trace)
