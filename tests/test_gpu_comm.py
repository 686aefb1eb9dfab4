"""The device data plane of sharded runs (csrc/comm.cu) on the GPU.

Ranks hold lane windows; their int64 partials (memo gains, CELF batch gains,
commit self-checks) are summed on the device.  One GPU is available, so
multi-rank runs use LOCAL ranks (threads of this process sharing the
device -- NCCL refuses two ranks per GPU) and the real NCCL backend is run
with one rank.  Every shard count must reproduce the reference's seeds,
seed gains, full dequeue trace and spread_se (tests/golden, made by the
reference; selection.py:115-149, propagation.py:371-390).
"""

import threading

import numpy as np
import pytest

from conftest import load_golden
from test_gpu_golden import build_graph

pytestmark = pytest.mark.gpu


def _shards(gpu, z, comms):
    from paper_2008_03095_b200.celf import lane_window
    from paper_2008_03095_b200.context import DeviceContext
    g = build_graph(gpu, z)
    randoms = gpu.SimulationRandoms(int(z["R"]), int(z["master_seed"]))
    table = gpu.build_hash_table(g)
    table.bind(g)
    ctxs = []
    for comm in comms:
        a, b, scored = lane_window(randoms.padded, randoms.num_scored, comm.rank, comm.size)
        c = DeviceContext(g, randoms.values[a:b], scored, a)
        c.propagate()
        c.attach_comm(comm)
        ctxs.append(c)
    return ctxs, randoms


def _run_ranks(ctxs, k):
    out, errs = [None] * len(ctxs), []

    def run(r):
        try:
            gains = ctxs[r].memoize(want_gains=True)          # summed over the ranks
            ctxs[r].celf_reset(None)
            out[r] = (gains,) + tuple(ctxs[r].celf_select_comm(k))
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(len(ctxs))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    return out


@pytest.mark.parametrize("shards", [1, 2, 3])
@pytest.mark.parametrize("name", ["er_mid_300", "er_pad20", "er_const1_r16", "cfg_c1", "kat_ties"])
def test_local_ranks_match_reference(gpu, name, shards):
    from paper_2008_03095_b200.celf import NativeComm
    z = load_golden(name)
    comms = NativeComm.local_group(shards, gpu.current_device() if hasattr(gpu, "current_device") else 0)
    ctxs, randoms = _shards(gpu, z, comms)
    out = _run_ranks(ctxs, int(z["k"]))
    per_sim = np.concatenate([c.per_sim() for c in ctxs])
    for gains, seeds, sg, trace in out:
        assert np.array_equal(gains, z["gains"])
        assert seeds.tolist() == z["seeds"].tolist()
        assert sg.tolist() == z["seed_gains"].tolist()
        assert np.array_equal(np.asarray(trace), z["trace"])
    R = randoms.num_scored
    se = 0.0 if R < 2 else float(per_sim.std(ddof=1) / np.sqrt(R))
    assert se == pytest.approx(float(z["spread_se"]), rel=1e-12, abs=1e-15)


def test_local_ranks_run_fused_on_config(gpu, orc):
    """C2 through run_fused itself, 2 LOCAL ranks: every rank returns the
    single-rank run's seeds, gains and trace, and the gathered labels/sizes
    and owned matrix of the sharded result equal the single-rank ones."""
    from paper_2008_03095_b200 import configs
    from paper_2008_03095_b200.celf import NativeComm
    g = configs.build("c2")
    one = gpu.run_fused(g, 10, num_simulations=256, master_seed=0)
    comms = NativeComm.local_group(2)
    g.device_graph()
    gpu.build_hash_table(g).bind(g)
    res, errs = [None, None], []

    def run(r):
        try:
            res[r] = gpu.run_fused(g, 10, num_simulations=256, master_seed=0, comm=comms[r])
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    for run in res:
        assert run.seeds == one.seeds
        assert run.selection.gains == one.selection.gains
        assert np.array_equal(run.selection.trace.array, one.selection.trace.array)
        assert run.spread_se == one.spread_se


def test_nccl_single_rank_matches_reference(gpu):
    """The NCCL backend itself (ncclCommInitRank with one rank, in-place
    ncclAllReduce on the context stream)."""
    import ctypes
    from paper_2008_03095_b200 import _lib
    from paper_2008_03095_b200._lib import check
    from paper_2008_03095_b200.celf import NativeComm
    lib = _lib.load()
    idbuf = (ctypes.c_uint8 * _lib.COMM_ID_BYTES)()
    check(lib.imx_comm_unique_id(idbuf))
    h = ctypes.c_void_p()
    check(lib.imx_comm_create(_lib.current_device(), 1, 0, idbuf, ctypes.byref(h)))
    comm = NativeComm(h, 0, 1)
    assert comm.allreduce(np.array([3, -4, 5])).tolist() == [3, -4, 5]
    for name in ("er_mid_300", "cfg_c2"):
        z = load_golden(name)
        ctxs, _ = _shards(gpu, z, [comm])
        (gains, seeds, sg, trace), = _run_ranks(ctxs, int(z["k"]))
        assert np.array_equal(gains, z["gains"])
        assert seeds.tolist() == z["seeds"].tolist()
        assert sg.tolist() == z["seed_gains"].tolist()
        assert np.array_equal(np.asarray(trace), z["trace"])
    comm.close()


def test_nccl_comm_from_torch_group(gpu, monkeypatch):
    """NativeComm.from_torch: the NCCL unique id travels through a
    torch.distributed group (one rank here), then the in-library NCCL
    communicator sums on the device."""
    import socket

    import torch
    import torch.distributed as dist
    from paper_2008_03095_b200 import _lib
    from paper_2008_03095_b200.celf import NativeComm
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    monkeypatch.setenv("MASTER_ADDR", "127.0.0.1")
    monkeypatch.setenv("MASTER_PORT", str(port))
    dev = _lib.current_device()
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", dev))
    try:
        comm = NativeComm.from_torch()
        assert (comm.rank, comm.size) == (0, 1)
        assert NativeComm.from_torch() is comm               # cached per group/device
        assert comm.allreduce(np.arange(5)).tolist() == [0, 1, 2, 3, 4]
        assert [p.tolist() for p in comm.allgather(np.array([7, 8]))] == [[7, 8]]
    finally:
        dist.destroy_process_group()
