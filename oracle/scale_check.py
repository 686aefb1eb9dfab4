"""Config-scale parity check of a device ``run_fused`` -- TEST INFRASTRUCTURE.

Used by tests/test_gpu_scale.py and by bench.py's ``parity`` field (outside
every timed region), never by the product package.

SURVEY 8(c).1-2: the full (n, R) matrices of C4/C5 are too large for the
dense restatement's time budget, so the check runs lane chunk by lane chunk:

* labels of every chunk [a, b) are copied from the device context
  (imx_copy_labels) and compared with ``oracle.uf_labels`` on X[a:b]
  (propagate reads only randoms.values[:width], propagation.py:269-279, so a
  chunk of X gives exactly those columns);
* sizes of every chunk (imx_copy_sizes) are compared with the oracle's
  component_sizes of the same chunk;
* the chunks' fresh-gain difference tables are summed and the reference's
  CELF heap is run on the exact fresh-gain table (oracle.SelectionCheck):
  initial gains, seeds, seed gains, the full dequeue trace, sigma and
  spread_se are compared with the device run;
* optionally, a window of lanes at each end is also compared with the dense
  min-label restatement (oracle.propagate), the primary oracle.
"""

from __future__ import annotations

import time

import numpy as np

import oracle


def config_host_graph(cfg):
    """(xadj, adj, weights) of a BASELINE config built on the host only --
    the repo's config generator restated in C (oracle.config_csr) and the
    config's weight scheme as apply_weights draws it (per-edge schemes: one
    draw per canonical slot in slot order, graph.py:251-259)."""
    from paper_2008_03095_b200 import configs
    from paper_2008_03095_b200.weights import parse_weight_scheme
    c = configs.CONFIGS[cfg]
    kind, n, m, draws, probs, cdf = configs._spec(cfg)
    xadj, adj = oracle.config_csr(kind, n, m, c.seed, draws, probs, cdf)
    scheme = parse_weight_scheme(c.weights)
    if hasattr(scheme, "p"):
        w = np.full(len(adj), float(scheme.p))
    else:
        src = oracle.sources(xadj)
        canon = np.flatnonzero(src < adj)
        rec = oracle.reciprocal(xadj, adj)
        draws = np.clip(np.random.default_rng(c.seed).normal(scheme.mean, scheme.std,
                                                              size=len(canon)), 0, 1)
        w = np.empty(len(adj))
        w[canon] = draws
        w[rec[canon]] = draws
    return xadj, adj, w


def host_sampler_inputs(g):
    """(xadj, adj, hashes, thr) of a Graph on the host; thr is an int when
    every slot has the same threshold (uniform schemes)."""
    xadj = np.asarray(g.xadj, np.int64)
    adj = np.asarray(g.adj, np.int32)
    w = np.asarray(g.weights, np.float64)
    hashes = oracle.hash_table(xadj, adj)
    if len(w) and bool((w == w[0]).all()):
        thr = int(oracle.thresholds(w[:1])[0])
    else:
        thr = oracle.thresholds(w, oracle.reciprocal(xadj, adj))
    return xadj, adj, hashes, thr


def check_fused_run(run, g, k, num_simulations, master_seed=0, chunk=None, dense_window=0,
                    nthreads=None, inputs=None):
    """Compare a single-context FusedRun with the oracle on every lane.
    Returns a report dict; ``ok`` is True when everything matched."""
    t0 = time.perf_counter()
    ctx = run._ctx
    xadj, adj, hashes, thr = inputs or host_sampler_inputs(g)
    X = oracle.randoms(num_simulations, master_seed)
    n, P = g.n, len(X)
    if chunk is None:                   # ~1 GB of int32 per chunk array
        chunk = max(8, min(P, (1 << 28) // max(n, 1) // 8 * 8))
    rep = {"lanes": P, "chunk": chunk, "labels": True, "sizes": True, "first_bad_lane": None}
    chk = oracle.SelectionCheck(n, k, np.asarray(run.seeds, np.int32), num_simulations)
    for a in range(0, P, chunk):
        b = min(P, a + chunk)
        want = oracle.uf_labels(xadj, adj, hashes, thr, X[a:b], nthreads)
        got = ctx.labels(a, b)
        if not np.array_equal(got, want):
            rep["labels"] = False
            bad = np.flatnonzero((got != want).any(axis=0))
            rep["first_bad_lane"] = rep["first_bad_lane"] or int(a + bad[0])
        del got
        sizes = chk.add_chunk(want, a, nthreads)
        if not np.array_equal(ctx.sizes(a, b), sizes):
            rep["sizes"] = False
        del want, sizes
    ref = chk.result()
    tr = np.asarray(run.selection.trace.array if hasattr(run.selection.trace, "array")
                    else run.selection.trace)
    gains = ctx.memoize(want_gains=True)
    rep.update({
        "gains": bool(np.array_equal(gains, ref["gains"])),
        "seeds": [int(s) for s in run.seeds] == ref["seeds"].tolist(),
        "seed_gains": [int(x) for x in run.selection.gains] == ref["seed_gains"].tolist(),
        "sigma": int(run.selection.sigma) == ref["sigma"],
        "trace": bool(tr.shape == ref["trace"].shape and np.array_equal(tr, ref["trace"])),
        "trace_records": int(len(ref["trace"])),
        "spread_se": float(run.spread_se) == float(ref["spread_se"]),
    })
    if dense_window:
        wins = sorted({(0, min(P, dense_window)), (max(0, P - dense_window), P)})
        ok = True
        for a, b in wins:
            want, _ = oracle.propagate(xadj, adj, hashes, thr, X[a:b], nthreads)
            ok &= bool(np.array_equal(ctx.labels(a, b), want))
        rep["dense_windows"] = [list(w) for w in wins]
        rep["dense_labels"] = ok
    keys = ("labels", "sizes", "gains", "seeds", "seed_gains", "sigma", "trace", "spread_se")
    rep["ok"] = all(rep[x] for x in keys) and rep.get("dense_labels", True)
    rep["check_s"] = round(time.perf_counter() - t0, 2)
    return rep
