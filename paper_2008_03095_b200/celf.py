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
in (-stale, id) order -- exactly R_t = {v : (-stale_v, v) <= (-fresh_u*, u*)}.
Round t therefore evaluates the top-priority vertex, then every vertex whose
stale key is at most that vertex's fresh key (a superset of R_t), and
replays R_t as refresh records before the commit record.
"""

from __future__ import annotations

import numpy as np

__all__ = ["LocalComm", "TorchComm", "select_rounds", "lane_window"]


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


def lane_window(padded: int, num_scored: int, rank: int, size: int):
    """Contiguous lane window [a, b) of rank and its number of scored lanes."""
    a = (padded * rank) // size
    b = (padded * (rank + 1)) // size
    scored = max(0, min(b, num_scored) - a)
    return a, b, scored


def _key_le(pa, va, pb, vb) -> bool:
    """(-pa, va) <= (-pb, vb)"""
    return pa > pb or (pa == pb and va <= vb)


def select_rounds(shard, comm, k: int, batch0: int = 64):
    """k seeds, their gains and the dequeue trace (T, 5) over a sharded
    CELF state.  ``shard`` offers celf_top / eval_gains / celf_collect /
    celf_eval_collected / celf_set_prio / commit (context.DeviceContext).

    Round t: evaluate the top-priority vertex; collect every vertex whose
    stale key is at most that fresh key (sorted by stale key, identical on
    every rank); evaluate it in doubling batches until the best fresh key is
    below the next stale key.  Each partial evaluation is allreduced."""
    seeds, gains, trace = [], [], []
    for t in range(k):
        g_top, v_top = shard.celf_top()
        if v_top < 0:
            raise AssertionError(f"no candidate left at round {t}")
        best_v, best_f = v_top, g_top
        if t > 0:
            f1 = int(comm.allreduce(shard.eval_gains(np.array([v_top], np.int32)))[0])
            best_f = f1
            ev_ids, ev_prio, ev_fresh = [v_top], [g_top], [f1]
            if f1 != g_top:
                ids, prio = shard.celf_collect(f1, v_top, v_top)
                lo, b = 0, batch0
                while lo < len(ids) and not _key_le(best_f, best_v, int(prio[lo]), int(ids[lo])):
                    hi = min(len(ids), lo + b)
                    fr = comm.allreduce(shard.celf_eval_collected(lo, hi))
                    for v, f in zip(ids[lo:hi].tolist(), fr.tolist()):
                        if _key_le(f, v, best_f, best_v):
                            best_v, best_f = v, f
                    ev_ids += ids[lo:hi].tolist()
                    ev_prio += prio[lo:hi].tolist()
                    ev_fresh += fr.tolist()
                    lo, b = hi, 2 * b
            ev = sorted((-p, v, f) for v, p, f in zip(ev_ids, ev_prio, ev_fresh)
                        if _key_le(p, v, best_f, best_v))
            for negp, v, f in ev:
                trace.append((v, -negp, f, 0, t))
            batch0 = max(64, len(ev))
            shard.celf_set_prio(np.array([v for _, v, _ in ev], np.int32),
                                np.array([f for _, _, f in ev], np.int64))
        got = int(comm.allreduce(np.array([shard.commit(best_v)], np.int64))[0])
        if got != best_f:
            raise AssertionError(f"committed gain {got} != evaluated {best_f} for vertex {best_v}")
        trace.append((best_v, best_f, best_f, 1, t))
        seeds.append(best_v)
        gains.append(best_f)
    return (np.asarray(seeds, np.int32), np.asarray(gains, np.int64),
            np.asarray(trace, np.int64).reshape(-1, 5))
