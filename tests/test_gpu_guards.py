"""Input guards on the caller-array entry points (GPU).

The reference indexes numpy arrays with caller labels (IndexError on a bad
label, selection.py:63-81) and runs a lazy heap that is exact for ANY
priorities (selection.py:128-147).  The device path must neither read nor
write out of bounds on bad labels, nor go wrong on priorities that are not
upper bounds of the gains.
"""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _ctx(gpu, n, width, ns=None):
    from paper_2008_03095_b200.context import DeviceContext, empty_graph
    return DeviceContext(empty_graph(n), np.zeros(width, np.int32), width if ns is None else ns)


@pytest.mark.parametrize("bad", [-1, 10, 1 << 30])
@pytest.mark.parametrize("with_sizes", [False, True])
def test_load_labels_rejects_out_of_range_labels(gpu, bad, with_sizes):
    labels = np.tile(np.arange(10, dtype=np.int32)[:, None], (1, 8))
    labels[3, 5] = bad
    sizes = np.ones_like(labels) if with_sizes else None
    ctx = _ctx(gpu, 10, 8)
    with pytest.raises(IndexError):
        ctx.load_labels(labels, sizes)
    with pytest.raises(ValueError):        # nothing usable was loaded
        ctx.memoize()


def test_load_labels_rejects_negative_sizes(gpu):
    labels = np.tile(np.arange(10, dtype=np.int32)[:, None], (1, 8))
    sizes = np.ones_like(labels)
    sizes[2, 1] = -4
    with pytest.raises(ValueError, match="negative"):
        _ctx(gpu, 10, 8).load_labels(labels, sizes)


def test_caller_labels_hub_histogram(gpu, orc):
    """k_hist_full's run-length aggregation: long runs of one label (a hub
    component) and ragged row counts give the oracle's sizes and gains."""
    rng = np.random.default_rng(5)
    n, W = 1000 + 7, 40
    labels = np.zeros((n, W), np.int32)
    for r in range(W):
        comp = rng.integers(0, 3, n)
        labels[:, r] = np.where(comp == 0, 0, np.arange(n))
        labels[0, r] = 0
    ctx = _ctx(gpu, n, W, 37)
    ctx.load_labels(labels)
    gains = ctx.memoize()
    sizes, want = orc.sizes_gains(labels, 37)
    assert np.array_equal(ctx.sizes(), sizes)
    assert np.array_equal(gains, want)


@pytest.mark.parametrize("name", ["er_mid_300", "er_big_1000", "kat_ties"])
def test_select_seeds_with_underestimating_priorities(gpu, orc, name):
    """Caller priorities below the true gains: the reference's heap commits
    the top stale entry at round 0 and refreshes lazily; the device path must
    give its exact seeds, gains and trace."""
    z = load_golden(name)
    labels, sizes = orc.run_fused(*_graph(orc, z), int(z["k"]), int(z["R"]), int(z["master_seed"]),
                                  nthreads=4)["labels"], None
    sizes, gains = orc.sizes_gains(labels, int(z["R"]))
    rng = np.random.default_rng(1)
    init = gains - rng.integers(0, np.maximum(gains, 1) + 1)           # some below, some equal
    init[rng.integers(0, len(init), 5)] += 10 ** 6                    # a few far above
    n = labels.shape[0]
    g = gpu.Graph.from_edges(n, z["edges"].astype(np.int64))
    res = gpu.select_seeds(g, labels, sizes, init, int(z["k"]), int(z["R"]))
    s, sg, tr, _ = orc.celf(labels, sizes, init, int(z["k"]), int(z["R"]))
    assert res.seeds == s.tolist()
    assert res.gains == sg.tolist()
    assert np.array_equal(res.trace.array, tr)


def _graph(orc, z):
    xadj, adj, _ = orc.csr_from_edges(int(z["n"]), z["edges"].astype(np.int64))
    w = z["weights"] if "weights" in z else np.full(len(adj), float(str(z["scheme"]).split(":")[1]))
    return xadj, adj, w


def test_celf_reset_refuses_priorities_below_the_memo(gpu, orc):
    z = load_golden("er_mid_300")
    labels = z["labels"]
    ctx = _ctx(gpu, labels.shape[0], labels.shape[1])
    ctx.load_labels(labels)
    gains = ctx.memoize()
    low = gains.copy()
    low[np.argmax(gains)] -= 1
    with pytest.raises(ValueError, match="upper bounds"):
        ctx.celf_reset(low)
    ctx.celf_reset(gains + 1)              # over-estimates are fine


@pytest.mark.parametrize("tile", ["64", "128"])
def test_wide_lane_tiles_with_fused_memo(gpu, tile, monkeypatch):
    """Lane tiles wider than 32 with the memo fused into the tiled
    compression: k_gains_tile sums every quad of a tile row, so the gains
    (and everything after them) stay the reference's."""
    monkeypatch.setenv("IMX_TILE_LANES", tile)
    z = load_golden("er_big_1000")
    from test_gpu_golden import build_graph
    g = build_graph(gpu, z)
    run = gpu.run_fused(g, int(z["k"]), num_simulations=int(z["R"]), master_seed=int(z["master_seed"]))
    assert run.seeds == z["seeds"].tolist()
    assert np.array_equal(run.selection.trace.array, z["trace"])


# ---- deferred weights (large host CSRs; forced on small ones) ----------------

def _deferred_graph(gpu, xadj, adj, w, pinned=False):
    if pinned:
        import torch

        def pin(a):
            t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
            out = t.numpy()
            out[...] = a
            return out
        xadj, adj, w = pin(xadj), pin(adj), pin(w)
    return gpu.Graph(xadj, adj, w, np.arange(len(xadj) - 1, dtype=np.int64))


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("case", ["uniform", "first_differs", "last_differs", "zero_first"])
def test_deferred_weights_speculation(gpu, orc, case, pinned, monkeypatch):
    """The weights of a large host CSR arrive after the propagate started on
    the speculative threshold of weights[0]; whatever the weights turn out to
    be, the result is the oracle's (the propagate reruns when the speculation
    fails)."""
    monkeypatch.setenv("IMX_LATE_WEIGHTS", "1")
    z = load_golden("er_big_1000")
    xadj, adj, _ = orc.csr_from_edges(int(z["n"]), z["edges"].astype(np.int64))
    w = np.full(len(adj), 0.05)
    rec = orc.reciprocal(xadj, adj)
    if case == "first_differs":
        w[[0, rec[0]]] = 0.3
    elif case == "last_differs":
        w[[-1, rec[-1]]] = 0.6
    elif case == "zero_first":
        w[[0, rec[0]]] = 0.0
    g = _deferred_graph(gpu, xadj, adj, w, pinned)
    run = gpu.run_fused(g, 5, num_simulations=40, master_seed=2)
    want = orc.run_fused(xadj, adj, w, 5, 40, 2, nthreads=4)
    assert np.array_equal(run.labels, want["labels"])
    assert run.seeds == want["seeds"].tolist()
    assert np.array_equal(run.selection.trace.array, want["trace"])
    assert np.array_equal(gpu.slot_thresholds(g), want["thr"])


def test_deferred_weights_asymmetric_csr_is_refused(gpu, monkeypatch):
    monkeypatch.setenv("IMX_LATE_WEIGHTS", "1")
    xadj = np.array([0, 2, 3, 4], np.int64)
    adj = np.array([1, 2, 0, 1], np.int32)          # 0-2 has no 2-0
    g = gpu.Graph(xadj, adj, np.full(4, 0.5), np.arange(3, dtype=np.int64))
    with pytest.raises(Exception, match="symmetric"):
        gpu.run_fused(g, 1, num_simulations=8)


def test_deferred_weights_unsorted_row_is_refused(gpu, monkeypatch):
    monkeypatch.setenv("IMX_LATE_WEIGHTS", "1")
    xadj = np.array([0, 2, 3, 4], np.int64)
    adj = np.array([2, 1, 0, 0], np.int32)          # row 0 not ascending
    g = gpu.Graph(xadj, adj, np.full(4, 0.5), np.arange(3, dtype=np.int64))
    with pytest.raises(Exception, match="symmetric"):
        gpu.run_fused(g, 1, num_simulations=8)


def test_deferred_weights_evaluate_and_reciprocal(gpu, orc, monkeypatch):
    """Consumers of the lazily built reciprocal slots on a deferred graph."""
    monkeypatch.setenv("IMX_LATE_WEIGHTS", "1")
    z = load_golden("er_mid_300")
    xadj, adj, _ = orc.csr_from_edges(int(z["n"]), z["edges"].astype(np.int64))
    g = _deferred_graph(gpu, xadj, adj, z["weights"])
    assert np.array_equal(g.reciprocal_slots, orc.reciprocal(xadj, adj))
    from paper_2008_03095_b200.evaluation import evaluate_counts
    got = evaluate_counts(g, np.array([1, 5, 9]), 300, 4)
    want = orc.evaluate_counts(xadj, adj, z["weights"], np.array([1, 5, 9]), 300, 4, nthreads=2)
    assert np.array_equal(got, want)


# ---- streamed CSR (very large pinned host CSRs; forced on small ones) ---------

def _stream_env(monkeypatch, hook, chunks="5", heavy=None):
    monkeypatch.setenv("IMX_LATE_WEIGHTS", "1")
    monkeypatch.setenv("IMX_STREAM_CSR", "1")
    monkeypatch.setenv("IMX_STREAM_CHUNKS", chunks)
    if hook:
        monkeypatch.setenv("IMX_HOOK", hook)
    if heavy:
        monkeypatch.setenv("IMX_SCAN_HEAVY", heavy)


@pytest.mark.parametrize("hook,heavy", [(None, None), ("scan", None), ("scan", "4"), ("pull", None), ("enum", None)])
@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("case", ["uniform", "last_differs"])
def test_streamed_csr_matches_oracle(gpu, orc, case, pinned, hook, heavy, monkeypatch):
    """imx_graph_from_csr returns before the adjacency is up; the scan's first
    pass runs on the chunks as they land (with and without heavy-row slices),
    every other sampler settles the structure first.  Results are the
    oracle's, also when the weight speculation fails afterwards."""
    _stream_env(monkeypatch, hook, heavy=heavy)
    z = load_golden("er_big_1000")
    xadj, adj, _ = orc.csr_from_edges(int(z["n"]), z["edges"].astype(np.int64))
    w = np.full(len(adj), 0.05)
    if case == "last_differs":
        rec = orc.reciprocal(xadj, adj)
        w[[-1, rec[-1]]] = 0.6
    g = _deferred_graph(gpu, xadj, adj, w, pinned)
    run = gpu.run_fused(g, 5, num_simulations=40, master_seed=2)
    want = orc.run_fused(xadj, adj, w, 5, 40, 2, nthreads=4)
    assert np.array_equal(run.labels, want["labels"])
    assert np.array_equal(run.sizes, want["sizes"])
    assert run.seeds == want["seeds"].tolist()
    assert np.array_equal(run.selection.trace.array, want["trace"])
    assert np.array_equal(gpu.slot_thresholds(g), want["thr"])


@pytest.mark.parametrize("chunks", ["1", "3", "16", "32"])
@pytest.mark.parametrize("name", ["cfg_c1", "cfg_c2"])
def test_streamed_csr_golden_configs(gpu, name, chunks, monkeypatch):
    """The benchmark graphs through the streamed build (C2 takes the scan
    sampler by rule, with isolated vertices and chunk cuts inside hub rows'
    neighbourhoods) against the reference's own outputs."""
    _stream_env(monkeypatch, None, chunks=chunks)
    z = load_golden(name)
    from test_gpu_golden import build_graph, check_array
    g0 = build_graph(gpu, z)
    g = _deferred_graph(gpu, np.asarray(g0.xadj), np.asarray(g0.adj), np.asarray(g0.weights), pinned=True)
    run = gpu.run_fused(g, int(z["k"]), num_simulations=int(z["R"]), master_seed=int(z["master_seed"]))
    check_array(z, "labels", run.labels)
    check_array(z, "sizes", run.sizes)
    assert run.seeds == z["seeds"].tolist()
    assert np.array_equal(run.selection.trace.array, z["trace"])
    # the graph's lazily built parts after a streamed build
    assert np.array_equal(g.reciprocal_slots, g0.reciprocal_slots)
    assert np.array_equal(gpu.build_hash_table(g).hashes, gpu.build_hash_table(g0).hashes)


@pytest.mark.parametrize("hook", [None, "scan"])
@pytest.mark.parametrize("bad,match", [
    ("asymmetric", "symmetric"), ("unsorted", "symmetric"), ("range", "outside"), ("offsets", "offsets")])
def test_streamed_csr_refuses_bad_input(gpu, bad, match, hook, monkeypatch):
    """What imx_graph_from_csr reports for a bad CSR surfaces from the
    streamed build too (at the latest when the structure is settled inside
    the propagate), and nothing is read out of bounds before."""
    _stream_env(monkeypatch, hook, chunks="2")
    xadj = np.array([0, 2, 3, 4], np.int64)
    adj = np.array([1, 2, 0, 0], np.int32)
    if bad == "asymmetric":
        adj = np.array([1, 2, 0, 1], np.int32)          # 0-2 has no 2-0
    elif bad == "unsorted":
        adj = np.array([2, 1, 0, 0], np.int32)
    elif bad == "range":
        adj = np.array([1, 7, 0, 0], np.int32)
    elif bad == "offsets":
        xadj = np.array([0, 3, 2, 4], np.int64)
    g = gpu.Graph(xadj, adj, np.full(4, 0.5), np.arange(3, dtype=np.int64))
    with pytest.raises(Exception, match=match):
        gpu.run_fused(g, 1, num_simulations=8)


# ---- CELF: seed-table batches evaluated by k_wide_tab_round --------------------

@pytest.mark.parametrize("name", ["er_mid_300", "er_big_1000", "er_pad20", "er_wc_r40", "cfg_c1", "cfg_c2"])
def test_wide_tab_round_forced(gpu, name, monkeypatch):
    """Every seed-table batch (rounds 1-4) leaves the persistent CELF kernel
    for the streaming kernel and the device-wide round finish (at scale only
    rounds that evaluate > 37 k candidates at once do): one listed seed with
    the table in registers, 2-4 listed seeds through L1, row quads that end
    inside a quad (R = 20).  Seeds, gains and the full trace stay the
    reference's."""
    monkeypatch.setenv("IMX_CELF_WIDE_OUT", "0")
    from test_gpu_golden import build_graph
    z = load_golden(name)
    g = build_graph(gpu, z)
    run = gpu.run_fused(g, int(z["k"]), num_simulations=int(z["R"]), master_seed=int(z["master_seed"]))
    assert run.seeds == z["seeds"].tolist()
    assert run.selection.gains == z["seed_gains"].tolist()
    assert np.array_equal(run.selection.trace.array, z["trace"])
    assert run.spread_se == pytest.approx(float(z["spread_se"]), rel=1e-12, abs=1e-15)


def test_deferred_speculation_guard_refuses_unconfirmed_results(gpu, orc, monkeypatch):
    """imx_spec_defer hands the check of the speculative threshold to the
    caller; a caller that forgets it still cannot read unconfirmed results:
    the getters settle the weights themselves and fail when the speculation
    did not hold, and a second propagate (on the settled thresholds) gives
    the oracle's labels."""
    monkeypatch.setenv("IMX_LATE_WEIGHTS", "1")
    z = load_golden("er_big_1000")
    xadj, adj, _ = orc.csr_from_edges(int(z["n"]), z["edges"].astype(np.int64))
    w = np.full(len(adj), 0.05)
    rec = orc.reciprocal(xadj, adj)
    w[[-1, rec[-1]]] = 0.6                       # weights[0]'s threshold is not every slot's
    g = _deferred_graph(gpu, xadj, adj, w, pinned=True)
    from paper_2008_03095_b200.context import DeviceContext
    X = gpu.SimulationRandoms(40, 2).values
    ctx = DeviceContext(g, X, 40)
    ctx.spec_defer(True)
    ctx.propagate()
    with pytest.raises(ValueError, match="speculative"):      # IMX_EINVAL, like "labels not computed"
        ctx.labels()
    assert ctx.spec_settle() is True             # settled by the guard; nothing pending any more
    ctx.propagate()
    want = orc.run_fused(xadj, adj, w, 5, 40, 2, nthreads=4)
    assert np.array_equal(ctx.labels()[:, :40], want["labels"][:, :40])
    # and the explicit protocol: settle says no, propagate again
    g2 = _deferred_graph(gpu, xadj, adj, w, pinned=True)
    ctx2 = DeviceContext(g2, X, 40)
    ctx2.spec_defer(True)
    ctx2.propagate()
    assert ctx2.spec_settle() is False
    ctx2.propagate()
    assert np.array_equal(ctx2.labels()[:, :40], want["labels"][:, :40])
    ctx.close()
    ctx2.close()
