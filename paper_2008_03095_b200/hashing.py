"""Direction-oblivious edge hashes and per-simulation random words.

Sampler semantics (reference hashing.py): undirected edge
{u, v} hashes to murmur3_x86_32(LE32(min) || LE32(max), seed 0) & 0x7FFFFFFF;
simulation r owns one 31-bit word X[r]; the edge is live in r iff
``(X[r] ^ hash) < int(w * H_MAX)`` (strict, signed 32-bit).  The per-slot
hash table and thresholds are produced by device kernels (K2) and are never
needed on the host by the fused pipeline: ``EdgeHashTable.hashes`` is copied
back only when someone reads it.
"""

from __future__ import annotations

import struct

import numpy as np

from . import _lib
from ._lib import check, ptr
from .graph import Graph

H_MAX = 2**31 - 1
LANE_WIDTH = 8
MURMUR_SEED = 0

__all__ = ["H_MAX", "LANE_WIDTH", "MURMUR_SEED", "murmur3_32", "EdgeHashTable",
           "build_hash_table", "SimulationRandoms", "sample_prob", "threshold",
           "lane_membership", "slot_thresholds"]

_M32 = 0xFFFFFFFF


def _rotl(x: int, r: int) -> int:
    return ((x << r) | (x >> (32 - r))) & _M32


def _scramble(k: int) -> int:
    return (_rotl((k * 0xCC9E2D51) & _M32, 15) * 0x1B873593) & _M32


def murmur3_32(key: bytes, seed: int = 0) -> int:
    """MurmurHash3 x86_32 of arbitrary bytes (host helper for known-answer
    checks; reference hashing.py:31-62)."""
    h = seed & _M32
    nblocks = len(key) // 4
    for (k,) in struct.iter_unpack("<I", key[: 4 * nblocks]):
        h = (_rotl(h ^ _scramble(k), 13) * 5 + 0xE6546B64) & _M32
    tail = key[4 * nblocks:]
    if tail:
        h ^= _scramble(int.from_bytes(tail, "little"))
    h ^= len(key)
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & _M32
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & _M32
    return h ^ (h >> 16)


def _murmur3_pair_array(lo, hi) -> np.ndarray:
    """Unmasked murmur3 of the 8-byte keys (lo[i], hi[i]) on the device
    (reference hashing.py:65-86)."""
    lo = np.ascontiguousarray(lo, dtype=np.uint32)
    hi = np.ascontiguousarray(hi, dtype=np.uint32)
    if lo.shape != hi.shape:
        raise ValueError("lo and hi must have the same shape")
    out = np.empty(lo.shape, dtype=np.uint32)
    _lib.require_device()
    check(_lib.load().imx_murmur3_pairs(_lib.current_device(), ptr(lo.reshape(-1)),
                                        ptr(hi.reshape(-1)), lo.size, ptr(out.reshape(-1))))
    return out


class EdgeHashTable:
    """Per-slot 31-bit hashes; reciprocal slots carry identical values
    (reference hashing.py:89-94).

    Built by ``build_hash_table`` the table lives on the device (inside the
    graph's device copy) and ``hashes`` is fetched lazily; constructed from an
    explicit array it is uploaded when a kernel needs it.
    """

    def __init__(self, hashes=None, h_max: int = H_MAX, *, _graph: Graph | None = None):
        self.h_max = h_max
        self._hashes = None if hashes is None else np.asarray(hashes, dtype=np.int32)
        self._graph = _graph

    @property
    def hashes(self) -> np.ndarray:
        if self._hashes is None:
            g = self._graph
            self.bind(g)
            out = np.empty(g.m, dtype=np.int32)
            check(_lib.load().imx_graph_hashes(g.device_graph().handle, ptr(out)))
            self._hashes = out
        return self._hashes

    def bind(self, g: Graph) -> None:
        """Make ``g``'s device copy sample with these hashes."""
        dg = g.device_graph()
        if self._graph is g:
            if dg.custom_hashes is not None:      # restore the computed table
                check(_lib.load().imx_graph_set_hashes(dg.handle, None))
                dg.custom_hashes = None
            return
        h = np.ascontiguousarray(self.hashes, dtype=np.int32)
        if h.shape != (g.m,):
            raise ValueError(f"hash table has {h.shape[0]} slots, graph has {g.m}")
        if dg.custom_hashes is not h:
            check(_lib.load().imx_graph_set_hashes(dg.handle, ptr(h)))
            dg.custom_hashes = h


def build_hash_table(g: Graph) -> EdgeHashTable:
    """Per-slot masked murmur3 of (min, max), computed on the device when the
    graph's CSR is built/uploaded (reference hashing.py:97-101)."""
    g.device_graph()
    return EdgeHashTable(_graph=g)


class SimulationRandoms:
    """One 31-bit random word per simulation (reference hashing.py:104-123).

    The words are numpy PCG64 draws -- ``default_rng(seed).integers(0, H_MAX,
    endpoint=True)`` over the padded count -- so they are prefix-stable and
    identical to the reference's for the same numpy version.  The count is
    padded to a multiple of LANE_WIDTH; padded lanes are propagated but not
    scored.
    """

    def __init__(self, count: int, master_seed: int = 0):
        if count < 1:
            raise ValueError(f"simulation count must be positive, got {count}")
        self.master_seed = int(master_seed)
        self.num_scored = int(count)
        padded = LANE_WIDTH * ((int(count) + LANE_WIDTH - 1) // LANE_WIDTH)
        words = np.random.default_rng(self.master_seed).integers(
            0, H_MAX, size=padded, endpoint=True, dtype=np.int64)
        self.values = words.astype(np.int32)

    @property
    def padded(self) -> int:
        return len(self.values)


def sample_prob(hash_value: int, xr: int) -> int:
    """Integer numerator of the sampling probability: X_r XOR hash."""
    return int(hash_value) ^ int(xr)


def threshold(w: float) -> int:
    """floor(w * H_MAX) for w in [0, 1] (reference hashing.py:135-138)."""
    if not 0.0 <= w <= 1.0:
        raise ValueError(f"weight {w} outside [0, 1]")
    return int(w * H_MAX)


def lane_membership(slot: int, r0: int, w: float, table: EdgeHashTable,
                    randoms: SimulationRandoms) -> int:
    """Bitmask of the LANE_WIDTH simulations r0.. in which ``slot`` is live
    (bit b <-> simulation r0 + b); reference hashing.py:141-150."""
    if r0 % LANE_WIDTH:
        raise ValueError(f"batch start {r0} not aligned to {LANE_WIDTH}")
    if r0 + LANE_WIDTH > randoms.padded:
        raise ValueError(f"batch [{r0}, {r0 + LANE_WIDTH}) beyond R")
    h = int(table.hashes[slot])
    t = threshold(w)
    mask = 0
    for b in range(LANE_WIDTH):
        if (int(randoms.values[r0 + b]) ^ h) < t:
            mask |= 1 << b
    return mask


def slot_thresholds(g: Graph, symmetrize: bool = True) -> np.ndarray:
    """Per-slot int32(int64(w * H_MAX)), max-symmetrized over reciprocal
    slots (reference hashing.py:153-165); computed on the device."""
    out = np.empty(g.m, dtype=np.int32)
    check(_lib.load().imx_graph_thresholds(g.device_graph().handle, 1 if symmetrize else 0,
                                           ptr(out), None))
    return out
