"""Seed-set evaluation on fresh worlds and the sampling-uniformity statistic
(reference evaluation.py:101-136, :143-190) on the device.

``evaluate_seeds`` returns the reference's (mean, se) bit for bit: the host
only derives the 128-bit PCG64 state of every chunk's stream from
``SeedSequence(rng_seed).spawn`` (numpy, a few microseconds per chunk); the
device reproduces every draw from those states (csrc/evaluation.cu), so the
per-world counts, and the mean / standard error computed from them with
numpy, equal the reference's.  Chunks of 4096 worlds are independent, so
under torch.distributed (>1 rank) each rank scores a contiguous range of
chunks and the counts are all-gathered in chunk order.

``sampling_cdf`` sorts the (hash ^ X) / H_MAX values on the device and
returns the exact KS distance and the numpy-rule histogram.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, ptr
from .graph import Graph
from .hashing import H_MAX, EdgeHashTable, SimulationRandoms

__all__ = ["evaluate_seeds", "evaluate_counts", "chunk_range", "SamplingCdf", "sampling_cdf", "write_cdf_tsv",
           "KS_UNIFORM_BOUND"]

_WORLD_CHUNK = 4096           # evaluation.py:29
_MAX_CDF_VALUES = 20_000_000  # evaluation.py:35
KS_UNIFORM_BOUND = 0.01       # evaluation.py:37
_M64 = (1 << 64) - 1


def _streams(rng_seed: int, nchunks: int) -> np.ndarray:
    """(nchunks, 4) uint64 {state_hi, state_lo, inc_hi, inc_lo} of the
    per-chunk PCG64 streams (evaluation.py:121-127)."""
    out = np.empty((nchunks, 4), np.uint64)
    for i, ss in enumerate(np.random.SeedSequence(rng_seed).spawn(nchunks)):
        st = np.random.default_rng(ss).bit_generator.state["state"]
        out[i] = (st["state"] >> 64, st["state"] & _M64, st["inc"] >> 64, st["inc"] & _M64)
    return out


def _check_seeds(g: Graph, seeds) -> np.ndarray:
    seeds = sorted({int(s) for s in seeds})
    if not seeds:
        raise ValueError("seed set must be nonempty")
    if any(not 0 <= s < g.n for s in seeds):
        raise ValueError("seed outside vertex range")
    return np.array(seeds, dtype=np.int32)


def chunk_range(nchunks: int, rank: int, size: int) -> tuple[int, int]:
    """Contiguous range [c0, c1) of world chunks scored by ``rank``."""
    return nchunks * rank // size, nchunks * (rank + 1) // size


def _device_counts(g: Graph, seeds: np.ndarray, streams: np.ndarray, worlds: int) -> np.ndarray:
    counts = np.empty(worlds, np.int64)
    _lib.require_device()
    st = np.ascontiguousarray(streams, dtype=np.uint64)
    check(_lib.load().imx_evaluate_seeds(g.device_graph().handle, ptr(seeds), len(seeds), worlds, ptr(st),
                                         _WORLD_CHUNK, ptr(counts)))
    return counts


def evaluate_counts(g: Graph, seeds, r_eval: int, rng_seed: int = 0, comm=None,
                    _score=_device_counts) -> np.ndarray:
    """Reached-set size of each of the ``r_eval`` fresh worlds (int64)."""
    s = _check_seeds(g, seeds)
    r_eval = int(r_eval)
    if r_eval < 1:
        raise ValueError(f"r_eval must be >= 1, got {r_eval}")
    if comm is None:
        from .pipeline import default_comm
        comm = default_comm()
    nch = -(-r_eval // _WORLD_CHUNK)
    streams = _streams(rng_seed, nch)
    c0, c1 = chunk_range(nch, comm.rank, comm.size)
    w0, w1 = c0 * _WORLD_CHUNK, min(r_eval, c1 * _WORLD_CHUNK)
    counts = _score(g, s, streams[c0:c1], w1 - w0) if w1 > w0 else np.empty(0, np.int64)
    if comm.size > 1:
        counts = np.concatenate(comm.allgather(counts))
    return counts


def evaluate_seeds(g: Graph, seeds, r_eval: int, rng_seed: int = 0, n_threads: int = 1,
                   comm=None, _score=_device_counts) -> tuple[float, float]:
    """Mean and standard error of the reached-set size over ``r_eval`` fresh
    worlds (evaluation.py:101-136); ``n_threads`` is accepted for API parity
    (the result never depends on it)."""
    counts = evaluate_counts(g, seeds, r_eval, rng_seed, comm, _score)
    r_eval = len(counts)
    mean = float(counts.mean())
    se = float(counts.std(ddof=1) / math.sqrt(r_eval)) if r_eval > 1 else 0.0
    return mean, se


@dataclass
class SamplingCdf:
    """Empirical CDF of hash sampling probabilities with its KS distance
    (evaluation.py:143-154)."""

    bin_uppers: np.ndarray
    cdf: np.ndarray
    ks_distance: float
    num_values: int

    @property
    def uniform_ok(self) -> bool:
        return self.ks_distance < KS_UNIFORM_BOUND


def sampling_cdf(g: Graph, table: EdgeHashTable, randoms: SimulationRandoms,
                 bins: int = 100) -> SamplingCdf:
    """Distribution of (X[r] ^ hash) / H_MAX over the canonical slots
    (strided down to ~20M values) and scored simulations
    (evaluation.py:157-183)."""
    if bins < 10:
        raise ValueError(f"need at least 10 bins, got {bins}")
    bins = int(bins)
    _lib.require_device()
    table.bind(g)
    dg = g.device_graph()
    me = g.num_undirected_edges
    scored = randoms.num_scored
    stride = max(1, math.ceil(me * scored / _MAX_CDF_VALUES))
    if me == 0 or scored == 0:   # the reference's max() over an empty array
        raise ValueError("zero-size array to reduction operation maximum which has no identity")
    edges = np.linspace(0.0, 1.0, bins + 1)     # np.histogram's uniform bin edges
    X = np.ascontiguousarray(randoms.values[:scored], dtype=np.int32)
    counts = np.empty(bins, np.int64)
    ks = ctypes.c_double()
    nv = ctypes.c_int64()
    check(_lib.load().imx_sampling_cdf(dg.handle, ptr(X), scored, stride, bins, ptr(edges), ptr(counts),
                                       ctypes.byref(ks), ctypes.byref(nv)))
    n_vals = int(nv.value)
    cdf = np.cumsum(counts) / n_vals
    uppers = np.arange(1, bins + 1) / bins
    return SamplingCdf(uppers, cdf, float(ks.value), n_vals)


def write_cdf_tsv(result: SamplingCdf, path) -> None:
    """Two-column TSV (bin_upper, cdf) (evaluation.py:186-190)."""
    with open(path, "w", encoding="utf-8") as fh:
        for upper, c in zip(result.bin_uppers, result.cdf):
            fh.write(f"{upper:.6f}\t{c:.8f}\n")
