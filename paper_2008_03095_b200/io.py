"""Graph file formats (reference graph.py:269-437): text edge lists and the
binary CSR cache ``INFCSR1``.

``load_edge_list`` parses with the native loader of libinfuser_b200
(``imx_edge_list_parse``, csrc/io.cpp: first-appearance id compaction,
first-occurrence dedupe, the reference's error kinds and line numbers) and
builds the CSR on the GPU (``Graph.from_edges``); the messages are formatted
here exactly as the reference formats them.  ``write_edge_list`` restates the
reference's round-trip ordering; ``save_csr`` / ``load_csr`` are the
reference's byte layout.  ``load_graph`` dispatches on the cache magic.
"""

from __future__ import annotations

import ctypes
import struct
from pathlib import Path

import numpy as np

from . import _lib
from ._lib import ConstraintError, GraphFormatError, check, ptr
from .graph import MAX_VERTICES, Graph

__all__ = ["load_edge_list", "write_edge_list", "save_csr", "load_csr", "load_graph", "CACHE_MAGIC"]

CACHE_MAGIC = b"INFCSR1\x00"   # graph.py:26
_ERR_TEXT = 1 << 16


def load_edge_list(path, directed_input: bool = False) -> Graph:
    """Whitespace-separated "u v [w]" edge list -> symmetric CSR
    (graph.py:273-330).  ``directed_input`` does not change the result (both
    directions are stored and duplicates collapse)."""
    edges, w, orig = _parse_edge_list(path)
    if len(orig) >= MAX_VERTICES:
        raise ConstraintError(f"{path}: {len(orig)} vertices exceed the 2^31 id limit")
    return Graph.from_edges(len(orig), edges, w, orig)


def _parse_edge_list(path):
    """(edges (k, 2) compact ids, weights (k,), orig_ids (n,)) of a text edge
    list, parsed natively (host code; no device needed)."""
    try:
        fh = open(path, "r", encoding="utf-8")
    except OSError as exc:
        raise GraphFormatError(f"cannot open {path}: {exc}") from exc
    fh.close()
    lib = _lib.load()
    h = ctypes.c_void_p()
    line, kind, aux = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int64()
    text = ctypes.create_string_buffer(_ERR_TEXT)
    rc = lib.imx_edge_list_parse(str(path).encode(), ctypes.byref(h), ctypes.byref(line), ctypes.byref(kind),
                                 ctypes.byref(aux), text, _ERR_TEXT)
    if rc != 0:
        _raise_parse_error(path, kind.value, line.value, aux.value, text.value.decode("utf-8", "replace"))
    try:
        n, k = ctypes.c_int64(), ctypes.c_int64()
        check(lib.imx_edge_list_dims(h, ctypes.byref(n), ctypes.byref(k)))
        edges = np.empty((k.value, 2), np.int64)
        w = np.empty(k.value, np.float64)
        orig = np.empty(n.value, np.int64)
        check(lib.imx_edge_list_copy(h, ptr(edges), ptr(w), ptr(orig)))
    finally:
        lib.imx_edge_list_free(h)
    return edges, w, orig


def _raise_parse_error(path, kind: int, lineno: int, aux: int, text: str):
    if kind == 1:
        raise GraphFormatError(f"{path}: line {lineno}: expected 'u v [w]', got {aux} fields")
    if kind == 2:
        raise GraphFormatError(f"{path}: line {lineno}: non-numeric field in {text!r}")
    if kind == 3:
        raise GraphFormatError(f"{path}: line {lineno}: weight {float(text)} outside [0, 1]")
    if kind == 4:
        raise GraphFormatError(f"{path}: no edges")
    if kind == 6:
        raise OverflowError(f"{path}: line {lineno}: vertex id beyond int64 in {text!r}")
    if kind == 7:
        raise ConstraintError(f"{path}: {MAX_VERTICES - 1} vertices exceed the 2^31 id limit")
    raise GraphFormatError(f"cannot open {path}")


def write_edge_list(g: Graph, path) -> None:
    """One "u v w" line per undirected edge in original ids, ordered so that
    reloading reproduces the same id compaction (graph.py:333-391)."""
    canon = g.canonical_slots
    src = g.sources[canon]
    dst = g.adj[canon]
    emitted = np.zeros(len(canon), dtype=bool)
    key_order = np.lexsort((dst, src))
    src_sorted = src[key_order]
    dst_sorted = dst[key_order]
    lines: list[str] = []
    introduced = 0

    def edge_index(u: int, v: int) -> int:
        lo = int(np.searchsorted(src_sorted, u, side="left"))
        hi = int(np.searchsorted(src_sorted, u, side="right"))
        j = lo + int(np.searchsorted(dst_sorted[lo:hi], v))
        return int(key_order[j]) if j < hi and dst_sorted[j] == v else -1

    def emit(i: int) -> None:
        nonlocal introduced
        u, v = int(src[i]), int(dst[i])
        lines.append(f"{g.orig_ids[u]} {g.orig_ids[v]} {float(g.weights[g.slot(u, v)])!r}")
        emitted[i] = True
        introduced = max(introduced, v + 1)

    for k in range(g.n):
        if k < introduced:
            continue
        row = g.neighbors(k)
        prior = row[row < k]
        if len(prior):
            emit(edge_index(int(prior.min()), k))
            introduced = max(introduced, k + 1)
            continue
        i = edge_index(k, k + 1) if k + 1 < g.n else -1
        if i < 0:
            break          # not a loader-produced ordering: sorted emission below
        emit(i)
    for i in key_order:
        if not emitted[i]:
            emit(int(i))
    Path(path).write_text("\n".join(lines) + "\n", encoding="utf-8")


def save_csr(g: Graph, path) -> None:
    """Magic, little-endian u64 n and m, then xadj (int64), adj (int32),
    weights (float64), orig_ids (int64) (graph.py:397-405)."""
    with open(path, "wb") as fh:
        fh.write(CACHE_MAGIC)
        fh.write(struct.pack("<QQ", g.n, g.m))
        fh.write(g.xadj.astype("<i8").tobytes())
        fh.write(g.adj.astype("<i4").tobytes())
        fh.write(g.weights.astype("<f8").tobytes())
        fh.write(g.orig_ids.astype("<i8").tobytes())


def load_csr(path) -> Graph:
    """Inverse of save_csr (graph.py:408-428); the CSR is uploaded to the GPU
    on first use."""
    try:
        blob = Path(path).read_bytes()
    except OSError as exc:
        raise GraphFormatError(f"cannot open {path}: {exc}") from exc
    if blob[:8] != CACHE_MAGIC:
        raise GraphFormatError(f"{path}: not a CSR cache (bad magic)")
    n, m = struct.unpack_from("<QQ", blob, 8)
    off = 24
    expect = 24 + 8 * (n + 1) + 4 * m + 8 * m + 8 * n
    if len(blob) != expect:
        raise GraphFormatError(f"{path}: truncated CSR cache")
    xadj = np.frombuffer(blob, "<i8", n + 1, off).astype(np.int64)
    off += 8 * (n + 1)
    adj = np.frombuffer(blob, "<i4", m, off).astype(np.int32)
    off += 4 * m
    weights = np.frombuffer(blob, "<f8", m, off).astype(np.float64)
    off += 8 * m
    orig = np.frombuffer(blob, "<i8", n, off).astype(np.int64)
    return Graph(xadj, adj, weights, orig)


def load_graph(path) -> Graph:
    """Either format through one entry: dispatch on the cache magic
    (graph.py:431-437)."""
    with open(path, "rb") as fh:
        head = fh.read(8)
    if head == CACHE_MAGIC:
        return load_csr(path)
    return load_edge_list(path)
