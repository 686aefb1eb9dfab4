"""End-to-end fused pipeline: hash, propagate, memoize, select (reference
pipeline.py:1-66), with every phase on the GPU.

``run_fused`` keeps the reference signature and ``FusedRun`` surface
(seeds, spread, spread_se, original_seed_ids, timings keys).  Labels and
sizes stay in device memory and are copied to the host only when
``FusedRun.labels`` / ``.sizes`` are read.  Under ``torch.distributed`` with
world size G > 1 the simulations are split into G contiguous lane windows,
one per rank; gains and CELF partial sums are combined with int64
allreduces (celf.py).
"""

from __future__ import annotations

import time

import numpy as np

from .celf import LocalComm, NativeComm, TorchComm, lane_window
from .context import DeviceContext
from .graph import Graph
from .hashing import EdgeHashTable, SimulationRandoms, build_hash_table
from .propagation import propagated_context
from .selection import SelectionResult, _check_k, result_from_context

__all__ = ["FusedRun", "run_fused", "default_comm"]


class FusedRun:
    """Everything a caller might want back from one fused selection run."""

    def __init__(self, graph: Graph, selection: SelectionResult, ctx: DeviceContext,
                 table: EdgeHashTable, randoms: SimulationRandoms, timings: dict, comm=None):
        self.graph = graph
        self.selection = selection
        self.table = table
        self.randoms = randoms
        self.timings = timings
        self._ctx = ctx
        self._comm = comm or LocalComm()
        self._labels = None
        self._sizes = None

    def _gather(self, local: np.ndarray) -> np.ndarray:
        if self._comm.size == 1:
            return local
        parts = self._comm.allgather(local.reshape(-1).astype(np.int64))
        n = self.graph.n
        return np.concatenate([p.reshape(n, -1) for p in parts], axis=1).astype(np.int32)

    @property
    def labels(self) -> np.ndarray:
        """(n, padded R) int32 min-id labels (copied from the device once)."""
        if self._labels is None:
            self._labels = self._gather(self._ctx.labels())
        return self._labels

    @property
    def sizes(self) -> np.ndarray:
        """(n, padded R) int32 component sizes indexed by label."""
        if self._sizes is None:
            self._sizes = self._gather(self._ctx.sizes())
        return self._sizes

    @property
    def seeds(self) -> list:
        return self.selection.seeds

    @property
    def spread(self) -> float:
        return self.selection.spread

    @property
    def spread_se(self) -> float:
        return self.selection.spread_se()

    def original_seed_ids(self) -> list:
        return [int(self.graph.orig_ids[s]) for s in self.selection.seeds]


def default_comm():
    """TorchComm when torch.distributed is initialised with >1 rank."""
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            return TorchComm()
    except ImportError:
        pass
    return LocalComm()


def native_comm(comm):
    """The device data plane for comm: itself if it is a NativeComm, an NCCL
    NativeComm for a torch.distributed NCCL group (IMX_NATIVE_COMM=0 keeps
    the torch allreduces), else None (gloo / single rank)."""
    import os
    if isinstance(comm, NativeComm):
        return comm
    if (isinstance(comm, TorchComm) and comm.size > 1 and comm.device.type == "cuda"
            and os.environ.get("IMX_NATIVE_COMM", "1") != "0"):
        return NativeComm.from_torch(comm.group)
    return None


def run_fused(g: Graph, k: int, num_simulations: int = 256, master_seed: int = 0,
              n_threads: int = 1, comm=None) -> FusedRun:
    """Select k seeds over ``num_simulations`` memoized implicit samples
    (reference pipeline.py:44-66).  ``n_threads`` is accepted for signature
    compatibility; ``comm`` (default: torch.distributed if initialised)
    splits the simulations across ranks."""
    comm = comm or default_comm()
    _check_k(k, g.n)
    timings: dict[str, float] = {}
    t = time.perf_counter()
    table = build_hash_table(g)
    randoms = SimulationRandoms(num_simulations, master_seed)
    timings["hash"] = time.perf_counter() - t

    t = time.perf_counter()
    a, b, scored = lane_window(randoms.padded, randoms.num_scored, comm.rank, comm.size)
    # a large host graph's weights may still be on the link: everything up to
    # the seeds runs on the speculative threshold and is checked afterwards
    native = native_comm(comm) if comm.size > 1 else None
    ctx, _ = propagated_context(g, table, randoms.values[a:b], scored, lane0=a, fuse_memo=True,
                                defer_spec=comm.size == 1 or native is not None)
    timings["propagate"] = time.perf_counter() - t

    if native is not None:
        ctx.attach_comm(native)           # gains summed over the ranks on the device

    def score():
        t = time.perf_counter()
        if comm.size == 1 or native is not None:
            ctx.memoize(want_gains=False)
        else:
            gains = comm.allreduce(ctx.memoize(want_gains=True))
        timings["memoize"] = timings.get("memoize", 0.0) + time.perf_counter() - t
        t = time.perf_counter()
        if comm.size == 1:
            ctx.celf_reset(None)
            out = ctx.celf_select(k)
        elif native is not None:
            ctx.celf_reset(None)
            out = ctx.celf_select_comm(k)
        else:
            ctx.celf_reset(gains)
            # the select_rounds loop, driven from native code with comm's allreduce
            out = ctx.celf_select_sharded(k, comm)
        timings["select"] = timings.get("select", 0.0) + time.perf_counter() - t
        return out

    seeds, gains_k, trace = score()
    if not ctx.spec_settle():
        # the weights were not uniform at weights[0]'s threshold: again, on the settled thresholds
        t = time.perf_counter()
        ctx.propagate()
        timings["propagate"] += time.perf_counter() - t
        seeds, gains_k, trace = score()
    t = time.perf_counter()
    selection = result_from_context(ctx, seeds, gains_k, trace, randoms.num_scored)
    if comm.size > 1:
        per_sim = np.concatenate(comm.allgather(ctx.per_sim()))
        selection.state._per_sim = per_sim
        selection.state._ctx = None
        selection.state._shard = (ctx, comm)
    timings["select"] += time.perf_counter() - t
    timings["total"] = sum(timings.values())
    return FusedRun(g, selection, ctx, table, randoms, timings, comm)
