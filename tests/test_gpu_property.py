"""Randomised parity: many small seeded graphs (isolated vertices, hubs,
paths, p in {0, 1, random}, widths that are not multiples of 32, k up to n)
through every sampler strategy and the whole pipeline vs the C oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def random_graph(rng):
    n = int(rng.integers(2, 160))
    kind = rng.integers(0, 4)
    if kind == 0:        # sparse random
        m = int(rng.integers(0, 3 * n))
        e = rng.integers(0, n, size=(m, 2))
    elif kind == 1:      # star + noise
        e = np.column_stack([np.zeros(n - 1, int), np.arange(1, n)])
        e = np.vstack([e, rng.integers(0, n, size=(n // 3, 2))])
    elif kind == 2:      # path with chords
        e = np.column_stack([np.arange(n - 1), np.arange(1, n)])
        e = np.vstack([e, rng.integers(0, n, size=(n // 5, 2))])
    else:                # dense-ish block + isolated tail
        h = max(2, n // 3)
        e = rng.integers(0, h, size=(4 * h, 2))
    e = e[e[:, 0] != e[:, 1]]
    lo, hi = np.minimum(e[:, 0], e[:, 1]), np.maximum(e[:, 0], e[:, 1])
    key = np.unique(lo * n + hi)
    e = np.column_stack([key // n, key % n]).astype(np.int64)
    p = rng.choice([0.0, 1.0, -1.0, -1.0, -1.0])
    w = rng.random(len(e)) if p < 0 else np.full(len(e), p)
    return n, e, w


@pytest.mark.parametrize("seed", range(24))
def test_random_graphs_match_oracle(gpu, orc, seed, monkeypatch):
    rng = np.random.default_rng(1000 + seed)
    n, e, w = random_graph(rng)
    g = gpu.Graph.from_edges(n, e, w)
    R = int(rng.integers(1, 300))
    k = int(rng.integers(1, n + 1))
    want = orc.run_fused(g.xadj, g.adj, g.weights, k, R, seed, nthreads=2)
    for mode in ("enum", "pull", "dense", "hybrid", "scan", None):
        if mode:
            monkeypatch.setenv("IMX_HOOK", mode)
        else:
            monkeypatch.delenv("IMX_HOOK", raising=False)
        run = gpu.run_fused(g, k, num_simulations=R, master_seed=seed)
        assert np.array_equal(run.labels, want["labels"]), mode          # (n, padded R)
        assert np.array_equal(run.sizes, want["sizes"]), mode
        assert [int(s) for s in run.seeds] == want["seeds"].tolist(), mode
        assert list(run.selection.gains) == want["seed_gains"].tolist(), mode
        assert np.array_equal(run.selection.trace.array, want["trace"]), mode
        assert run.spread_se == pytest.approx(want["spread_se"], rel=1e-12, abs=0)


@pytest.mark.parametrize("seed", range(12))
def test_random_evaluate_matches_oracle(gpu, orc, seed):
    from paper_2008_03095_b200.evaluation import evaluate_counts
    rng = np.random.default_rng(5000 + seed)
    n, e, w = random_graph(rng)
    g = gpu.Graph.from_edges(n, e, w)
    seeds = rng.integers(0, n, size=int(rng.integers(1, 12)))
    r_eval = int(rng.choice([1, 7, 4095, 4096, 4097, 9000]))
    got = evaluate_counts(g, seeds, r_eval, seed)
    want = orc.evaluate_counts(g.xadj, g.adj, g.weights, seeds, r_eval, seed, nthreads=2)
    assert np.array_equal(got, want)


def hub_on_top_graph(rng):
    """Hubs with the LARGEST ids (long smaller-neighbour prefixes): the pull
    sampler splits such rows into slices (heavy rows) by default."""
    n = int(rng.integers(300, 700))
    parts = [rng.integers(0, n, size=(2 * n, 2))]
    for h in range(n - 3, n):
        nb = np.flatnonzero(rng.random(h) < 0.6)
        parts.append(np.column_stack([nb, np.full(len(nb), h)]))
    e = np.vstack(parts)
    e = e[e[:, 0] != e[:, 1]]
    lo, hi = np.minimum(e[:, 0], e[:, 1]), np.maximum(e[:, 0], e[:, 1])
    key = np.unique(lo * n + hi)
    e = np.column_stack([key // n, key % n]).astype(np.int64)
    return n, e, rng.random(len(e)) * 0.3


@pytest.mark.parametrize("seed", range(6))
def test_heavy_rows_match_oracle(gpu, orc, seed, monkeypatch):
    """Pull passes with heavy-row slices (default slice length, and 1-slot
    slices) through the whole pipeline vs the oracle."""
    rng = np.random.default_rng(7000 + seed)
    n, e, w = hub_on_top_graph(rng)
    g = gpu.Graph.from_edges(n, e, w)
    R = int(rng.choice([24, 100, 256, 300]))
    k = int(rng.integers(1, 12))
    want = orc.run_fused(g.xadj, g.adj, g.weights, k, R, seed, nthreads=2)
    for mode, heavy in ((None, None), ("pull", None), ("pull", "1"), ("hybrid", "3"), ("pull", "0")):
        for var, val in (("IMX_HOOK", mode), ("IMX_PULL_HEAVY", heavy)):
            if val is None:
                monkeypatch.delenv(var, raising=False)
            else:
                monkeypatch.setenv(var, val)
        run = gpu.run_fused(g, k, num_simulations=R, master_seed=seed)
        tag = (mode, heavy)
        assert np.array_equal(run.labels, want["labels"]), tag
        assert np.array_equal(run.sizes, want["sizes"]), tag
        assert [int(s) for s in run.seeds] == want["seeds"].tolist(), tag
        assert np.array_equal(run.selection.trace.array, want["trace"]), tag


@pytest.mark.parametrize("seed", range(6))
def test_scan_heavy_rows_match_oracle(gpu, orc, seed, monkeypatch):
    """The bucketed pull forest (uniform thresholds) with heavy-row slices of
    1, 3 and 512 slots and with splitting off, through the whole pipeline."""
    rng = np.random.default_rng(9000 + seed)
    n, e, _ = hub_on_top_graph(rng)
    p = float(rng.choice([0.003, 0.02, 0.2, 0.9]))
    g = gpu.Graph.from_edges(n, e, p)
    R = int(rng.choice([8, 24, 100, 256, 1100, 2100]))
    k = int(rng.integers(1, 12))
    want = orc.run_fused(g.xadj, g.adj, g.weights, k, R, seed, nthreads=2)
    monkeypatch.setenv("IMX_HOOK", "scan")
    for heavy in (None, "1", "3", "0"):
        if heavy is None:
            monkeypatch.delenv("IMX_SCAN_HEAVY", raising=False)
        else:
            monkeypatch.setenv("IMX_SCAN_HEAVY", heavy)
        run = gpu.run_fused(g, k, num_simulations=R, master_seed=seed)
        assert np.array_equal(run.labels, want["labels"]), heavy
        assert np.array_equal(run.sizes, want["sizes"]), heavy
        assert [int(s) for s in run.seeds] == want["seeds"].tolist(), heavy
        assert np.array_equal(run.selection.trace.array, want["trace"]), heavy
