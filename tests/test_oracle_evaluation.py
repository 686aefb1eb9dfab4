"""CPU: the evaluation oracle (oracle.c PCG64 worlds, numpy sampling_cdf) is
pinned to the reference's own outputs (tests/golden/eval_*, cdf_*, made by
make_golden_eval.py), and the product's chunk sharding of evaluate_seeds is
exercised over 2 gloo ranks with the oracle standing in for the device."""

from __future__ import annotations

import hashlib
import os
import socket

import numpy as np
import pytest

from conftest import golden_graph, golden_names, load_golden

EVAL = golden_names("eval_")
CDF = golden_names("cdf_")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_fixtures_present():
    assert len(EVAL) >= 7 and len(CDF) >= 4


@pytest.mark.parametrize("name", EVAL)
def test_oracle_evaluate_matches_reference(orc, name):
    z = load_golden(name)
    xadj, adj, w = golden_graph(z)
    if "cfg" in z:
        assert _sha(adj) == str(z["adj_sha"]) and _sha(w) == str(z["weights_sha"])
    counts = orc.evaluate_counts(xadj, adj, w, z["seeds"], int(z["r_eval"]), int(z["rng_seed"]))
    assert np.array_equal(counts, z["counts"])
    mean, se = orc.evaluate_seeds(xadj, adj, w, z["seeds"], int(z["r_eval"]), int(z["rng_seed"]))
    assert (mean, se) == (float(z["mean"]), float(z["se"]))


def test_oracle_evaluate_thread_invariant(orc):
    z = load_golden("eval_er1000")
    a = orc.evaluate_counts(z["xadj"], z["adj"], z["weights"], z["seeds"], 3000, 7, nthreads=1)
    b = orc.evaluate_counts(z["xadj"], z["adj"], z["weights"], z["seeds"], 3000, 7, nthreads=4)
    assert np.array_equal(a, b)


def test_pcg_streams_match_numpy(orc):
    # the per-chunk states reproduce numpy's draws (evaluation.py:121-127)
    st = orc.pcg_streams(3, 3 * 4096)
    M = 0x2360ED051FC65DA44385DF649FCCF645
    for i, ss in enumerate(np.random.SeedSequence(3).spawn(3)):
        want = np.random.default_rng(ss).random(4)
        s = (int(st[i, 0]) << 64) | int(st[i, 1])
        inc = (int(st[i, 2]) << 64) | int(st[i, 3])
        got = []
        for _ in range(4):
            s = (s * M + inc) & ((1 << 128) - 1)
            rot = s >> 122
            x = ((s >> 64) ^ s) & ((1 << 64) - 1)
            x = ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)
            got.append((x >> 11) * 2.0**-53)
        assert got == list(want)


@pytest.mark.parametrize("name", CDF)
def test_oracle_sampling_cdf_matches_reference(orc, name):
    z = load_golden(name)
    if "cfg" in z:
        from paper_2008_03095_b200 import configs
        c = configs.CONFIGS[str(z["cfg"])]
        xadj, adj, _ = orc.csr_from_edges(c.n, configs.edges(str(z["cfg"])))
        assert _sha(adj) == str(z["adj_sha"])
    else:
        xadj, adj = z["xadj"], z["adj"]
    h = orc.hash_table(xadj, adj)
    if bool(z["broken"]):
        h[:] = 0
    up, cdf, ks, k = orc.sampling_cdf(xadj, adj, h, z["X"], int(z["num_scored"]), int(z["bins"]))
    assert k == int(z["num_values"])
    assert ks == float(z["ks"])
    assert np.array_equal(cdf, z["cdf"]) and np.array_equal(up, z["bin_uppers"])


def test_chunk_range_partition():
    from paper_2008_03095_b200.evaluation import chunk_range
    for nch in (1, 2, 3, 7, 64):
        for size in (1, 2, 3, 8):
            parts = [chunk_range(nch, r, size) for r in range(size)]
            assert parts[0][0] == 0 and parts[-1][1] == nch
            assert all(parts[i][1] == parts[i + 1][0] for i in range(size - 1))


# ---- 2-rank gloo: chunk sharding + gather of evaluate_seeds ----------------

class _G:
    """Host-only stand-in for Graph (n + CSR) so the product's sharding logic
    runs without a device; the oracle scores each rank's chunks."""

    def __init__(self, z):
        self.xadj, self.adj, self.weights = golden_graph(z)
        self.n = len(self.xadj) - 1


def _oracle_score(g, seeds, streams, worlds):
    import oracle
    return oracle.evaluate_counts(g.xadj, g.adj, g.weights, seeds, worlds, streams=streams, nthreads=2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, name, out_dir):
    import torch.distributed as dist
    from paper_2008_03095_b200.celf import TorchComm
    from paper_2008_03095_b200.evaluation import evaluate_seeds
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        z = load_golden(name)
        mean, se = evaluate_seeds(_G(z), z["seeds"], int(z["r_eval"]), int(z["rng_seed"]),
                                  comm=TorchComm(), _score=_oracle_score)
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.array([mean, se]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["eval_er1000", "eval_er200"])
def test_two_rank_gloo_evaluate_matches_reference(tmp_path, name):
    import torch.multiprocessing as mp
    mp.start_processes(_rank_main, args=(2, _free_port(), name, str(tmp_path)), nprocs=2,
                       join=True, start_method="spawn")
    z = load_golden(name)
    for rank in range(2):
        mean, se = np.load(tmp_path / f"rank{rank}.npy")
        assert (float(mean), float(se)) == (float(z["mean"]), float(z["se"]))
