"""Device context: one lane window of the simulation set on one GPU.

Thin owner of an ``imx_ctx`` handle (include/infuser_b200.h).  A context
holds the label matrix L[n][W], the component counts, the CELF state and the
per-lane covered totals of lanes [lane0, lane0 + W) for the graph it was
created on.  Every method is a single C-ABI call; the context is also the
per-rank "shard" the multi-GPU CELF driver (celf.py) talks to.
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _lib
from ._lib import MODE_NAMES, PropStats, Timings, check, ptr

# int (*)(int64_t *buf, int64_t n, void *user): imx_allreduce_fn
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_int64, ctypes.c_void_p)

__all__ = ["DeviceContext", "empty_graph"]

_EMPTY = {}


def empty_graph(n: int):
    """Edgeless device graph on n vertices: the host for contexts that only
    receive labels (memoization / CELF on caller-provided arrays)."""
    from .graph import Graph
    g = Graph(np.zeros(n + 1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float64),
              np.arange(n, dtype=np.int64))
    return g


def _take_trace(handle) -> np.ndarray:
    """The (T, 5) trace as a zero-copy view of the library's pinned buffer,
    returned to the library's pinned cache when the array is collected."""
    lib = _lib.load()
    p, n = ctypes.c_void_p(), ctypes.c_int64()
    check(lib.imx_celf_trace_take(handle, ctypes.byref(p), ctypes.byref(n)))
    if not p.value:
        return np.empty((0, 5), np.int64)
    buf = (ctypes.c_int64 * (5 * n.value)).from_address(p.value)
    weakref.finalize(buf, lib.imx_host_free, p.value)
    return np.frombuffer(buf, dtype=np.int64).reshape(n.value, 5)


class DeviceContext:
    def __init__(self, graph, X: np.ndarray, num_scored: int, lane0: int = 0):
        X = np.ascontiguousarray(X, dtype=np.int32)
        if X.ndim != 1 or len(X) < 1:
            raise ValueError("need at least one simulation word")
        self.graph = graph                    # keeps the device graph alive
        self.dg = graph.device_graph()
        self.n = graph.n
        self.width = len(X)
        self.num_scored = int(num_scored)
        self.lane0 = int(lane0)
        h = ctypes.c_void_p()
        check(_lib.load().imx_create(self.dg.handle, ptr(X), self.width, self.num_scored,
                                     ctypes.byref(h)))
        self.handle = h

    def close(self):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            try:
                _lib.load().imx_destroy(h)
            except Exception:
                pass

    __del__ = close

    # -- K3 ---------------------------------------------------------------------
    def propagate(self, verify: bool = False, stats: bool = False):
        """Run the fused sample + CC; returns (sweeps, changed, label_sums, modes)
        when ``stats`` else None."""
        if not stats:
            check(_lib.load().imx_propagate(self.handle, 1 if verify else 0, None))
            return None
        cap = 8
        changed = np.zeros(cap, np.int64)
        sums = np.zeros(cap, np.int64)
        modes = np.zeros(cap, np.int32)
        st = PropStats(0, cap, changed.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                       sums.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                       modes.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
        check(_lib.load().imx_propagate(self.handle, 1 if verify else 0, ctypes.byref(st)))
        k = min(st.sweeps, cap)
        return (st.sweeps, changed[:k].tolist(), sums[:k].tolist(),
                [MODE_NAMES[int(x)] for x in modes[:k]])

    def spec_defer(self, on: bool = True):
        """Let memo and CELF run while a large host graph's weights are still
        uploading; the caller must check ``spec_settle()`` afterwards."""
        check(_lib.load().imx_spec_defer(self.handle, 1 if on else 0))

    def spec_settle(self) -> bool:
        """Wait for the graph's weights; False when the results so far stand
        on a speculative threshold that did not hold (propagate again)."""
        held = ctypes.c_int32(1)
        check(_lib.load().imx_spec_settle(self.handle, ctypes.byref(held)))
        return bool(held.value)

    # -- K4/K5 ------------------------------------------------------------------
    def set_fuse_memo(self, on: bool = True):
        """Sum the gains inside the next propagations' tiled compression."""
        check(_lib.load().imx_set_fuse_memo(self.handle, 1 if on else 0))

    def memoize(self, want_gains: bool = True):
        out = np.empty(self.n, np.int64) if want_gains else None
        check(_lib.load().imx_memoize(self.handle, ptr(out)))
        return out

    def load_labels(self, labels: np.ndarray, sizes: np.ndarray | None = None):
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        if sizes is not None:
            sizes = np.ascontiguousarray(sizes, dtype=np.int32)
            if sizes.shape != labels.shape:
                raise ValueError(f"sizes shape {sizes.shape} != labels shape {labels.shape}")
        try:
            check(_lib.load().imx_load_labels(self.handle, ptr(labels), ptr(sizes),
                                              labels.shape[1] if labels.ndim == 2 else self.width))
        except ValueError as e:
            if "label outside" in str(e):     # the reference's numpy gather raises IndexError
                raise IndexError(str(e)) from None
            raise

    def labels(self, r0: int = 0, r1: int | None = None) -> np.ndarray:
        r1 = self.width if r1 is None else r1
        out = np.empty((self.n, r1 - r0), np.int32)
        check(_lib.load().imx_copy_labels(self.handle, r0, r1, ptr(out)))
        return out

    def sizes(self, r0: int = 0, r1: int | None = None) -> np.ndarray:
        r1 = self.width if r1 is None else r1
        out = np.empty((self.n, r1 - r0), np.int32)
        check(_lib.load().imx_copy_sizes(self.handle, r0, r1, ptr(out)))
        return out

    # -- K6-K8 (the CELF shard interface) ----------------------------------------
    def celf_reset(self, prio: np.ndarray | None = None):
        p = None if prio is None else np.ascontiguousarray(prio, dtype=np.int64)
        check(_lib.load().imx_celf_reset(self.handle, ptr(p)))

    def celf_top(self):
        g, v = ctypes.c_int64(), ctypes.c_int32()
        check(_lib.load().imx_celf_top(self.handle, ctypes.byref(g), ctypes.byref(v)))
        return int(g.value), int(v.value)

    def celf_prefix(self, lo: int, hi: int):
        """Evaluate order[lo, hi): (ids, stale prio of order[lo, hi+1) clipped,
        partial fresh gains of order[lo, hi), current order length)."""
        cnt = max(0, hi - lo)
        ids = np.empty(cnt + 1, np.int32)
        pr = np.empty(cnt + 1, np.int64)
        fr = np.empty(cnt, np.int64)
        ln = ctypes.c_int64()
        check(_lib.load().imx_celf_prefix(self.handle, int(lo), int(hi), ptr(ids), ptr(pr), ptr(fr),
                                          ctypes.byref(ln)))
        length = ln.value
        h = max(lo, min(hi, length))
        f = min(h + 1, length)
        return ids[: max(0, f - lo)], pr[: max(0, f - lo)], fr[: h - lo], length

    def celf_advance(self, k: int, u: int, ids, prio) -> int:
        """Commit u, drop order[0, k), merge (ids, prio) back; partial gain of u."""
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        prio = np.ascontiguousarray(prio, dtype=np.int64)
        g = ctypes.c_int64()
        check(_lib.load().imx_celf_advance(self.handle, int(k), int(u), ptr(ids), ptr(prio), len(ids),
                                           ctypes.byref(g)))
        return int(g.value)

    def eval_gains(self, cand) -> np.ndarray:
        cand = np.ascontiguousarray(cand, dtype=np.int32)
        out = np.empty(len(cand), np.int64)
        check(_lib.load().imx_eval_gains(self.handle, ptr(cand), len(cand), ptr(out)))
        return out

    def commit(self, u: int) -> int:
        g = ctypes.c_int64()
        check(_lib.load().imx_commit(self.handle, int(u), ctypes.byref(g)))
        return int(g.value)

    def celf_select(self, k: int):
        """Single-context CELF loop: (seeds, gains, trace records (T, 5))."""
        lib = _lib.load()
        seeds = np.empty(k, np.int32)
        gains = np.empty(k, np.int64)
        tl = ctypes.c_int64()
        check(lib.imx_celf_select(self.handle, int(k), ptr(seeds), ptr(gains), ctypes.byref(tl)))
        return seeds, gains, _take_trace(self.handle)

    def celf_select_sharded(self, k: int, comm):
        """The CELF loop over this context's lane shard with the per-batch
        int64 sums over ranks done by ``comm.allreduce`` (celf.select_rounds
        semantics, driven from native code): (seeds, gains, trace (T, 5))."""
        lib = _lib.load()
        seeds = np.empty(k, np.int32)
        gains = np.empty(k, np.int64)
        tl = ctypes.c_int64()
        err = []

        def reduce(buf, n, _user):
            try:
                a = np.ctypeslib.as_array(buf, shape=(n,))
                a[:] = comm.allreduce(a.copy())
                return 0
            except BaseException as e:          # surfaced after the call
                err.append(e)
                return 1

        cb = ALLREDUCE_FN(reduce)
        rc = lib.imx_celf_select_sharded(self.handle, int(k), ctypes.cast(cb, ctypes.c_void_p), None,
                                         ptr(seeds), ptr(gains), ctypes.byref(tl))
        if err:
            raise err[0]
        check(rc)
        return seeds, gains, _take_trace(self.handle)

    def attach_comm(self, comm) -> None:
        """Sum this context's partials (memo gains, CELF batches) over the
        ranks of ``comm`` (a NativeComm) on the device."""
        self._comm = comm                      # keeps the communicator alive
        check(_lib.load().imx_ctx_attach_comm(self.handle, None if comm is None else comm.handle))

    def celf_select_comm(self, k: int):
        """CELF over the lane shards of the attached communicator:
        (seeds, gains, trace (T, 5)); every rank calls it."""
        lib = _lib.load()
        seeds = np.empty(k, np.int32)
        gains = np.empty(k, np.int64)
        tl = ctypes.c_int64()
        check(lib.imx_celf_select_comm(self.handle, int(k), ptr(seeds), ptr(gains), ctypes.byref(tl)))
        return seeds, gains, _take_trace(self.handle)

    def per_sim(self) -> np.ndarray:
        out = np.empty(self.num_scored, np.int64)
        check(_lib.load().imx_per_sim(self.handle, ptr(out)))
        return out

    def owned_bits(self) -> np.ndarray:
        cw = max(1, (self.num_scored + 31) // 32)
        out = np.empty((self.n, cw), np.uint32)
        check(_lib.load().imx_copy_owned(self.handle, ptr(out)))
        return out

    def owned(self) -> np.ndarray:
        """SeedState.owned as an (n, num_scored) bool matrix."""
        bits = self.owned_bits()
        unpacked = np.unpackbits(bits.view(np.uint8), axis=1, bitorder="little")
        return unpacked[:, : self.num_scored].astype(bool)

    # -- measurement --------------------------------------------------------------
    def timings(self) -> dict:
        t = Timings()
        check(_lib.load().imx_get_timings(self.handle, ctypes.byref(t)))
        return {f: getattr(t, f) for f, _ in Timings._fields_}

    def bench_propagate(self, reps: int, flush_l2: bool = True) -> dict:
        vals = [ctypes.c_float() for _ in range(4)]
        check(_lib.load().imx_bench_propagate(self.handle, int(reps), 1 if flush_l2 else 0,
                                              *[ctypes.byref(v) for v in vals]))
        return dict(zip(("total_ms", "hook_ms", "compress_ms", "init_ms"),
                        (v.value for v in vals)))
