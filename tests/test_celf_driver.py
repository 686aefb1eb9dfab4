"""Host logic of the sharded CELF driver (celf.select_rounds), CPU-only.

The per-rank device context is replaced by a numpy shard with the same
interface (test double); single-rank and 2-rank gloo runs must reproduce the
oracle's seeds, gains and full dequeue trace (which the oracle reproduces
from the reference, tests/test_oracle_golden.py).
"""

import os
import socket

import numpy as np
import pytest

from conftest import load_golden


class NumpyShard:
    """Lanes [a, b) of a label/size matrix; same CELF interface as
    DeviceContext (celf_top / celf_prefix / celf_advance)."""

    def __init__(self, labels, sizes, a, b, num_scored, prio):
        self.L = np.ascontiguousarray(labels[:, a:b])
        self.S = np.ascontiguousarray(sizes[:, a:b])
        self.ns = max(0, min(b, num_scored) - a)
        self.n = labels.shape[0]
        prio = np.asarray(prio, np.int64)
        ids = np.arange(self.n)
        order = np.lexsort((ids, -prio))
        self.order = [(int(prio[v]), int(v)) for v in order]   # sorted by (-prio, id)
        self.owned = np.zeros((self.n, self.ns), bool)
        self.per_sim = np.zeros(self.ns, np.int64)
        self.cols = np.arange(self.ns)

    def _fresh(self, ids):
        lu = self.L[np.asarray(ids, np.int64)][:, : self.ns]
        return np.where(self.owned[lu, self.cols], 0, self.S[lu, self.cols]).sum(axis=1).astype(np.int64)

    @property
    def num_scored(self):
        return self.ns

    def owned_bits(self):
        """The covered bitmap as DeviceContext.owned_bits returns it."""
        cw = max(1, (self.ns + 31) // 32)
        packed = np.packbits(self.owned, axis=1, bitorder="little")
        out = np.zeros((self.n, 4 * cw), np.uint8)
        out[:, : packed.shape[1]] = packed
        return out.view(np.uint32)

    def celf_top(self):
        if not self.order:
            return 0, -1
        return self.order[0]

    def celf_prefix(self, lo, hi):
        length = len(self.order)
        h = max(lo, min(hi, length))
        f = min(h + 1, length)
        ids = np.array([v for _, v in self.order[lo:f]], np.int32)
        pr = np.array([p for p, _ in self.order[lo:f]], np.int64)
        return ids, pr, self._fresh(ids[: h - lo]), length

    def celf_advance(self, k, u, ids, prio):
        lu = self.L[u, : self.ns]
        new = ~self.owned[lu, self.cols]
        gain = int(self.S[lu, self.cols][new].sum())
        self.per_sim[new] += self.S[lu, self.cols][new]
        self.owned[lu, self.cols] = True
        rest = self.order[k:] + [(int(p), int(v)) for v, p in zip(ids, prio)]
        self.order = sorted(rest, key=lambda pv: (-pv[0], pv[1]))
        return gain


def _case(name):
    z = load_golden(name)
    return z["labels"], z["sizes"], z["gains"], int(z["R"]), int(z["k"]), z


@pytest.mark.parametrize("name", ["er_mid_300", "er_big_1000", "er_const015_r32", "er_pad20",
                                  "er_const1_r16", "kat_path3", "kat_ties"])
def test_single_rank_driver_reproduces_reference_trace(name):
    from paper_2008_03095_b200.celf import LocalComm, select_rounds
    labels, sizes, gains, R, k, z = _case(name)
    shard = NumpyShard(labels, sizes, 0, labels.shape[1], R, gains)
    seeds, sg, trace = select_rounds(shard, LocalComm(), k, batch0=4)
    assert seeds.tolist() == z["seeds"].tolist()
    assert sg.tolist() == z["seed_gains"].tolist()
    assert np.array_equal(trace, z["trace"])


def test_lane_window_partition():
    from paper_2008_03095_b200.celf import lane_window
    for padded, scored, size in [(24, 20, 2), (1024, 1024, 8), (128, 128, 3), (8, 5, 4)]:
        wins = [lane_window(padded, scored, r, size) for r in range(size)]
        assert wins[0][0] == 0 and wins[-1][1] == padded
        assert all(wins[i][1] == wins[i + 1][0] for i in range(size - 1))
        assert sum(w[2] for w in wins) == scored


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, name, out_dir):
    import torch.distributed as dist
    from paper_2008_03095_b200.celf import TorchComm, gather_owned, lane_window, select_rounds
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        labels, sizes, _, R, k, _ = _case(name)
        a, b, scored = lane_window(labels.shape[1], R, rank, world)
        # partial initial gains, combined with the allreduce as run_fused does
        part = NumpyShard(labels, sizes, a, b, R, np.zeros(labels.shape[0], np.int64))
        comm = TorchComm()
        lu = part.L[:, : part.ns]
        local = part.S[lu, np.arange(part.ns)].sum(axis=1).astype(np.int64)
        gains = comm.allreduce(local)
        shard = NumpyShard(labels, sizes, a, b, R, gains)
        seeds, sg, trace = select_rounds(shard, comm, k, batch0=8)
        per_sim = np.concatenate(comm.allgather(shard.per_sim))
        owned = gather_owned(shard, comm)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), seeds=seeds, sg=sg, trace=trace,
                 gains=gains, per_sim=per_sim, owned=owned)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["er_mid_300", "er_pad20"])
def test_two_rank_gloo_driver_matches_single_rank(tmp_path, name):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.start_processes(_rank_main, args=(2, port, name, str(tmp_path)), nprocs=2,
                       join=True, start_method="spawn")
    labels, sizes, gains, R, k, z = _case(name)
    for rank in range(2):
        got = np.load(tmp_path / f"rank{rank}.npz")
        assert np.array_equal(got["gains"], z["gains"])
        assert got["seeds"].tolist() == z["seeds"].tolist()
        assert got["sg"].tolist() == z["seed_gains"].tolist()
        assert np.array_equal(got["trace"], z["trace"])
        assert float(got["per_sim"].std(ddof=1) / np.sqrt(R)) == pytest.approx(float(z["spread_se"]))
        # SeedState.owned of a sharded run: every rank sees all lanes
        want = np.zeros((labels.shape[0], R), bool)
        for u in z["seeds"].tolist():
            want[labels[u, :R], np.arange(R)] = True
        assert np.array_equal(got["owned"], want)


def test_native_comm_is_only_used_for_nccl_groups():
    """run_fused's data-plane choice: gloo groups and single ranks keep the
    host path; NativeComm objects are used as given."""
    from paper_2008_03095_b200.celf import LocalComm, NativeComm
    from paper_2008_03095_b200.pipeline import native_comm
    assert native_comm(LocalComm()) is None
    fake = NativeComm(None, 0, 2)
    assert native_comm(fake) is fake
