"""Round-based exact CELF across lane shards (multi-GPU driver).

With the simulations split over G ranks, every rank owns the labels, sizes
and covered bitmaps of its lane window, and every marginal gain is a sum of
per-rank partial sums.  The decision logic below is the same as the
single-context loop in csrc/cc.cu (imx_celf_select); it only inserts an
integer allreduce after each partial evaluation.  Because the priorities are
replicated and every reduction is an exact int64 sum, all ranks take
identical decisions.

Exactness: on one fixed sample family marginal gains are
submodular, so the reference's lazy heap (selection.py:131-147) commits in
round t the vertex u* minimising (-fresh, id) over V\\S, after refreshing --
in (-stale, id) order -- exactly R_t = {v : (-stale_v, v) <= (-fresh_u*, u*)},
which is a prefix of the non-seeds sorted by stale key.
"""

from __future__ import annotations

import numpy as np

__all__ = ["LocalComm", "TorchComm", "NativeComm", "select_rounds", "lane_window", "gather_owned"]


class LocalComm:
    """Single-rank communicator: allreduce is the identity."""

    rank = 0
    size = 1

    def allreduce(self, x: np.ndarray) -> np.ndarray:
        return np.asarray(x, dtype=np.int64)

    def allgather(self, x: np.ndarray) -> list:
        return [np.asarray(x)]


class TorchComm:
    """int64 sums over ``torch.distributed`` (NCCL on GPUs, gloo on CPUs)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        backend = dist.get_backend(group)
        self.device = (torch.device("cuda", torch.cuda.current_device())
                       if backend == "nccl" else torch.device("cpu"))

    def allreduce(self, x: np.ndarray) -> np.ndarray:
        t = self.torch.from_numpy(np.ascontiguousarray(x, dtype=np.int64)).to(self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy()

    def allgather(self, x: np.ndarray) -> list:
        x = np.ascontiguousarray(x, dtype=np.int64)
        cnt = self.allreduce_counts(len(x))
        width = int(max(cnt)) if len(cnt) else 0
        buf = np.zeros(width, np.int64)
        buf[: len(x)] = x
        t = self.torch.from_numpy(buf).to(self.device)
        parts = [self.torch.empty_like(t) for _ in range(self.size)]
        self.dist.all_gather(parts, t, group=self.group)
        return [p.cpu().numpy()[: int(c)] for p, c in zip(parts, cnt)]

    def allreduce_counts(self, k: int) -> np.ndarray:
        v = np.zeros(self.size, np.int64)
        v[self.rank] = k
        return self.allreduce(v)


class NativeComm:
    """The library's device data plane for a sharded run (csrc/comm.cu):
    partial sums are added on the GPU, in place, on the context's stream.

    ``from_torch()`` builds an NCCL communicator over a torch.distributed
    group (rank 0's NCCL unique id is broadcast through the group);
    ``local_group(n)`` builds n ranks that are threads of this process on one
    device (the test double: NCCL refuses two ranks per GPU)."""

    _cache: dict = {}

    def __init__(self, handle, rank: int, size: int, group=None):
        self.handle = handle
        self.rank = int(rank)
        self.size = int(size)
        self._group = group                  # a LOCAL group outlives its comms

    @classmethod
    def from_torch(cls, group=None, device: int | None = None) -> "NativeComm":
        import ctypes
        import torch.distributed as dist
        from . import _lib
        from ._lib import check
        rank, size = dist.get_rank(group), dist.get_world_size(group)
        if device is None:
            device = _lib.current_device()
        key = (id(group), rank, size, device)
        if key in cls._cache:
            return cls._cache[key]
        idbuf = (ctypes.c_uint8 * _lib.COMM_ID_BYTES)()
        if rank == 0:
            check(_lib.load().imx_comm_unique_id(idbuf))
        obj = [bytes(idbuf)]
        dist.broadcast_object_list(obj, src=0, group=group)
        idbuf = (ctypes.c_uint8 * _lib.COMM_ID_BYTES).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        check(_lib.load().imx_comm_create(int(device), size, rank, idbuf, ctypes.byref(h)))
        comm = cls(h, rank, size)
        cls._cache[key] = comm
        return comm

    @classmethod
    def local_group(cls, nranks: int, device: int = 0) -> list:
        import ctypes
        from . import _lib
        from ._lib import check
        lib = _lib.load()
        grp = ctypes.c_void_p()
        check(lib.imx_local_group_create(int(nranks), ctypes.byref(grp)))
        owner = _LocalGroupOwner(grp)
        out = []
        for r in range(nranks):
            h = ctypes.c_void_p()
            check(lib.imx_comm_create_local(grp, r, int(device), ctypes.byref(h)))
            out.append(cls(h, r, nranks, owner))
        return out

    def allreduce(self, x: np.ndarray) -> np.ndarray:
        from . import _lib
        from ._lib import check, ptr
        a = np.ascontiguousarray(x, dtype=np.int64).copy()
        check(_lib.load().imx_comm_allreduce(self.handle, ptr(a), len(a)))
        return a

    def allgather(self, x: np.ndarray) -> list:
        """Through allreduce: every rank writes its slot of a zero buffer."""
        x = np.ascontiguousarray(x, dtype=np.int64).reshape(-1)
        cnt = np.zeros(self.size, np.int64)
        cnt[self.rank] = len(x)
        cnt = self.allreduce(cnt)
        off = np.concatenate([[0], np.cumsum(cnt)])
        buf = np.zeros(int(off[-1]), np.int64)
        buf[off[self.rank]:off[self.rank + 1]] = x
        buf = self.allreduce(buf)
        return [buf[off[r]:off[r + 1]] for r in range(self.size)]

    def close(self):
        from . import _lib
        h, self.handle = self.handle, None
        if h:
            _lib.load().imx_comm_destroy(h)


class _LocalGroupOwner:
    def __init__(self, grp):
        self.grp = grp

    def __del__(self):
        try:
            from . import _lib
            _lib.load().imx_local_group_destroy(self.grp)
        except Exception:
            pass


def gather_owned(ctx, comm) -> np.ndarray:
    """SeedState.owned (n, num_scored) of a sharded run: every rank's covered
    bitmap over its lane window (imx_copy_owned), all-gathered and
    concatenated along the lanes in rank order (= lane order)."""
    bits = ctx.owned_bits()                                    # (n, ceil(ns_local/32)) uint32
    n = bits.shape[0]
    counts = comm.allgather(np.array([ctx.num_scored], np.int64))
    parts = comm.allgather(bits.astype(np.int64).reshape(-1))
    out = []
    for p, c in zip(parts, counts):
        ns = int(c[0])
        if ns == 0:
            continue
        b = np.asarray(p, np.int64).astype(np.uint32).reshape(n, -1)
        out.append(np.unpackbits(b.view(np.uint8), axis=1, bitorder="little")[:, :ns].astype(bool))
    return np.concatenate(out, axis=1) if out else np.zeros((n, 0), bool)


def lane_window(padded: int, num_scored: int, rank: int, size: int):
    """Contiguous lane window [a, b) of rank and its number of scored lanes."""
    a = (padded * rank) // size
    b = (padded * (rank + 1)) // size
    scored = max(0, min(b, num_scored) - a)
    return a, b, scored


def _key_le(pa, va, pb, vb) -> bool:
    """(-pa, va) <= (-pb, vb)"""
    return pa > pb or (pa == pb and va <= vb)


def _lex_best(ids: np.ndarray, gains: np.ndarray):
    """(gain, id) of the lexicographic best of a batch: max gain, then min id."""
    g = gains.max()
    return int(g), int(ids[gains == g].min())


def select_rounds(shard, comm, k: int, batch0: int = 64):
    """k seeds, their gains and the dequeue trace (T, 5) over a sharded CELF
    state.  ``shard`` offers celf_top / celf_prefix / celf_advance
    (context.DeviceContext); every partial gain is allreduced.

    Round t >= 1 evaluates prefixes of the stale-key order in doubling
    batches until the best fresh key is below the next stale key; the
    refreshed vertices are the prefix whose stale key is at most the
    winner's fresh key, replayed as refresh records, then the winner commits
    and the others go back into the order with their fresh keys.  The
    per-round host work is vectorised (numpy), so a round costs its device
    calls and allreduces, not a Python loop over the refreshed prefix."""
    seeds, gains, trace = [], [], []
    pending = None              # (local commit gain, expected, vertex) checked with the next allreduce

    def check(total):
        if total != pending[1]:
            raise AssertionError(f"committed gain {total} != evaluated {pending[1]} for vertex {pending[2]}")

    for t in range(k):
        if t == 0:
            best_f, best_v = shard.celf_top()
            if best_v < 0:
                raise AssertionError("no candidate left at round 0")
            kr = 1
            back_ids = np.empty(0, np.int32)
            back_prio = np.empty(0, np.int64)
        else:
            lo, hi = 0, batch0
            best_v, best_f = -1, -1
            ids_l, prio_l, fresh_l = [], [], []
            while True:
                i, p, f_part, length = shard.celf_prefix(lo, hi)
                if length == 0:
                    raise AssertionError(f"no candidate left at round {t}")
                if pending is not None:     # last round's commit check rides along
                    f = comm.allreduce(np.append(np.asarray(f_part, np.int64), pending[0]))
                    check(int(f[-1]))
                    pending = None
                    f = f[:-1]
                else:
                    f = comm.allreduce(f_part)
                h = min(hi, length)
                bi = np.asarray(i[: h - lo], np.int64)
                bf = np.asarray(f, np.int64)
                if len(bi):
                    g_b, v_b = _lex_best(bi, bf)
                    if best_v < 0 or _key_le(g_b, v_b, best_f, best_v):
                        best_v, best_f = v_b, g_b
                ids_l.append(bi)
                prio_l.append(np.asarray(p[: h - lo], np.int64))
                fresh_l.append(bf)
                if h >= length:
                    break
                if _key_le(best_f, best_v, int(p[h - lo]), int(i[h - lo])):
                    break                       # nothing unevaluated can win
                lo, hi = h, h + max(batch0, h)
            ids = np.concatenate(ids_l)
            prio = np.concatenate(prio_l)
            fresh = np.concatenate(fresh_l)
            # the order is sorted by (-prio, id): the refreshed vertices are the
            # prefix whose stale key is at most the winner's fresh key
            le = (prio > best_f) | ((prio == best_f) & (ids <= best_v))
            kr = int(np.argmin(le)) if not le.all() else len(le)
            rec = np.empty((kr, 5), np.int64)
            rec[:, 0], rec[:, 1], rec[:, 2], rec[:, 3], rec[:, 4] = ids[:kr], prio[:kr], fresh[:kr], 0, t
            trace.append(rec)
            keep = ids[:kr] != best_v
            bi, bg = ids[:kr][keep], fresh[:kr][keep]
            # back into the order sorted by (-fresh, id): one argsort of the
            # packed key fresh * 2^32 + (2^32 - 1 - id) when gains fit 31 bits
            if len(bg) and bg.max() < (1 << 31):
                o = np.argsort(-((bg << 32) | (0xFFFFFFFF - bi)), kind="stable")
            else:
                o = np.lexsort((bi, -bg))
            back_ids = bi[o].astype(np.int32)
            back_prio = bg[o]
            batch0 = max(64, kr)
        local = shard.celf_advance(kr, best_v, back_ids, back_prio)
        if t == k - 1:                  # no later evaluation allreduce to ride on
            pending = (local, best_f, best_v)
            check(int(comm.allreduce(np.array([local], np.int64))[0]))
            pending = None
        else:
            pending = (local, best_f, best_v)
        trace.append(np.array([[best_v, best_f, best_f, 1, t]], np.int64))
        seeds.append(best_v)
        gains.append(best_f)
    tr = np.concatenate(trace) if trace else np.empty((0, 5), np.int64)
    return np.asarray(seeds, np.int32), np.asarray(gains, np.int64), tr.reshape(-1, 5)
