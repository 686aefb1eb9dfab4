"""Undirected weighted graphs in CSR form, built and kept on the GPU.

Mirrors the reference ``infmax.graph`` surface that the hot path touches
(``Graph``, ``Graph.from_edges``, ``sources``, ``canonical_slots``,
``reciprocal_slots``, ``slot``, ``with_weights``; graph.py:37-155 of the
reference).  Weight schemes live in ``weights.py``.  Every undirected edge {u, v} occupies two directed
slots, so ``m == 2 * number_of_undirected_edges`` exactly as in the
reference.

The CSR builder is the device kernel K1 (``imx_graph_from_edges``: radix sort
of (src, dst) keys, duplicate/self-loop/range validation, offsets by binary
search); the reciprocal-slot map is a device kernel too.  A Graph keeps a
handle to its device copy so the propagate/memo/CELF kernels reuse it without
another upload.
"""

from __future__ import annotations

import ctypes
from functools import cached_property

import numpy as np

from . import _lib
from ._lib import ConstraintError, GraphFormatError, check, ptr

MAX_VERTICES = 2**31

__all__ = ["MAX_VERTICES", "ConstraintError", "GraphFormatError", "Graph", "DeviceGraph"]


class DeviceGraph:
    """Owner of one ``imx_graph`` handle (device-resident CSR + slot tables)."""

    def __init__(self, handle, device: int):
        self.handle = handle
        self.device = device
        self.custom_hashes = None   # host array uploaded over the computed hashes

    def __del__(self):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            try:
                _lib.load().imx_graph_destroy(h)
            except Exception:
                pass

    def dims(self):
        n, m2 = ctypes.c_int64(), ctypes.c_int64()
        check(_lib.load().imx_graph_dims(self.handle, ctypes.byref(n), ctypes.byref(m2)))
        return n.value, m2.value


class Graph:
    """Symmetric CSR adjacency of an undirected weighted graph.

    Attributes follow the reference (graph.py:37-60): ``xadj`` int64 (n+1),
    ``adj`` int32 (m), ``weights`` float64 (m), ``orig_ids`` int64 (n).
    """

    def __init__(self, xadj, adj, weights, orig_ids, _device_graph=None):
        self.xadj = np.asarray(xadj, dtype=np.int64)
        self.adj = np.asarray(adj, dtype=np.int32)
        self.weights = np.asarray(weights, dtype=np.float64)
        self.orig_ids = np.asarray(orig_ids, dtype=np.int64)
        self._dev = _device_graph

    # -- sizes ---------------------------------------------------------------
    @property
    def n(self) -> int:
        return len(self.xadj) - 1

    @property
    def m(self) -> int:
        return len(self.adj)

    @property
    def num_undirected_edges(self) -> int:
        return self.m // 2

    # -- derived slot data ---------------------------------------------------
    @cached_property
    def degrees(self) -> np.ndarray:
        return np.diff(self.xadj)

    @cached_property
    def sources(self) -> np.ndarray:
        """Source vertex of every slot (graph.py:75-78)."""
        return np.repeat(np.arange(self.n, dtype=np.int32), self.degrees)

    @cached_property
    def canonical_slots(self) -> np.ndarray:
        """Slot indices with source < neighbor (graph.py:80-83)."""
        return np.flatnonzero(self.sources < self.adj)

    @cached_property
    def reciprocal_slots(self) -> np.ndarray:
        """reciprocal_slots[i] is the slot of (v, u) given slot i is (u, v)
        (graph.py:85-99); computed on the device by binary search of u in
        row v.  Raises GraphFormatError if the adjacency is not symmetric."""
        dg = self.device_graph()
        out = np.empty(self.m, dtype=np.int64)
        check(_lib.load().imx_graph_reciprocal(dg.handle, ptr(out)))
        return out

    def neighbors(self, v: int) -> np.ndarray:
        return self.adj[self.xadj[v]: self.xadj[v + 1]]

    def neighbor_weights(self, v: int) -> np.ndarray:
        return self.weights[self.xadj[v]: self.xadj[v + 1]]

    def slot(self, u: int, v: int) -> int:
        """Index of directed slot (u, v); KeyError if the edge is absent."""
        row = self.neighbors(u)
        k = int(np.searchsorted(row, v))
        if k == len(row) or row[k] != v:
            raise KeyError(f"no edge ({u}, {v})")
        return int(self.xadj[u]) + k

    def with_weights(self, weights: np.ndarray) -> "Graph":
        """Same topology, new per-slot weights (graph.py:112-119)."""
        w = np.asarray(weights, dtype=np.float64)
        if w.shape != (self.m,):
            raise ValueError(f"expected {self.m} weights, got {w.shape}")
        if w.size and (w.min() < 0.0 or w.max() > 1.0):
            raise ConstraintError("weights must lie in [0, 1]")
        out = Graph(self.xadj, self.adj, w, self.orig_ids)
        for name in ("degrees", "sources", "canonical_slots"):
            if name in self.__dict__:
                out.__dict__[name] = self.__dict__[name]
        return out

    # -- device copy -----------------------------------------------------------
    def device_graph(self) -> DeviceGraph:
        """The device-resident CSR (uploaded on first use)."""
        if self._dev is None:
            _lib.require_device()
            h = ctypes.c_void_p()
            dev = _lib.current_device()
            w = np.ascontiguousarray(self.weights)
            check(_lib.load().imx_graph_from_csr(
                dev, self.n, self.m, ptr(np.ascontiguousarray(self.xadj)),
                ptr(np.ascontiguousarray(self.adj)), ptr(w), ctypes.byref(h)))
            self._dev = DeviceGraph(h, dev)
        return self._dev

    def drop_device(self) -> None:
        """Release the device copy (the next kernel call re-uploads it)."""
        self._dev = None

    @classmethod
    def from_edges(cls, n, edges, weights=1.0, orig_ids=None) -> "Graph":
        """Build a CSR graph from distinct undirected edges on 0..n-1 on the
        GPU (graph.py:124-155): self-loops, duplicates and out-of-range
        endpoints are rejected with the reference's messages; ``weights`` is
        a scalar or one value per undirected edge, copied to both directions."""
        if n < 0 or n >= MAX_VERTICES:
            raise ConstraintError(f"vertex count {n} outside [0, 2^31)")
        e = np.asarray(list(edges) if not isinstance(edges, np.ndarray) else edges,
                       dtype=np.int64).reshape(-1, 2)
        e = np.ascontiguousarray(e)
        k = len(e)
        w = np.asarray(weights, dtype=np.float64)
        w_edge = None
        w_scalar = 0.0
        if w.ndim == 0:
            w_scalar = float(w)
        else:
            w_edge = np.ascontiguousarray(np.broadcast_to(w, (k,)), dtype=np.float64)
        _lib.require_device()
        dev = _lib.current_device()
        h = ctypes.c_void_p()
        check(_lib.load().imx_graph_from_edges(dev, int(n), ptr(e), k, ptr(w_edge),
                                               w_scalar, ctypes.byref(h)))
        dg = DeviceGraph(h, dev)
        xadj = np.empty(int(n) + 1, dtype=np.int64)
        adj = np.empty(2 * k, dtype=np.int32)
        ww = np.empty(2 * k, dtype=np.float64)
        check(_lib.load().imx_graph_get_csr(h, ptr(xadj), ptr(adj), ptr(ww)))
        if orig_ids is None:
            orig_ids = np.arange(int(n), dtype=np.int64)
        return cls(xadj, adj, ww, np.asarray(orig_ids, dtype=np.int64), dg)
