"""The reference's own hot-path tests, re-run against the CUDA package.

Ported from the reference suite (tests/test_propagation.py,
tests/test_selection.py, tests/test_pipeline.py, tests/test_hashing.py,
tests/test_acceptance.py criteria 1, 2, 5, 6).  The reference's explicit-world
oracles (BFS labels, MixGreedy) are replaced by the CPU oracle, which is pinned
to the reference in tests/test_oracle_golden.py.  Tests that monkeypatch the
reference's numpy sweep internals (test_all_sweep_shapes_agree) or time its
thread pool have no meaning here; their device counterpart is
test_gpu_golden.py::test_every_sampler_strategy_reaches_the_reference_fixpoint.
"""

import csv
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCHEMES = ["const:0.15", "uniform:0.02,0.5", "normal:0.25,0.15", "wc"]


def make_graph(imx, edges, n=None, weights=1.0):
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if n is None:
        n = int(edges.max()) + 1
    return imx.Graph.from_edges(n, edges, weights)


def weighted_er(imx, n, deg, scheme, graph_seed=0, weight_seed=0):
    from paper_2008_03095_b200.generators import er_edges
    m = int(round(n * deg / 2))
    g = imx.Graph.from_edges(n, er_edges(n, m, graph_seed))
    return imx.apply_weights(g, imx.parse_weight_scheme(scheme), rng_seed=weight_seed)


def oracle_labels(orc, g, randoms, width=None):
    X = randoms.values[: (randoms.padded if width is None else width)]
    thr = orc.thresholds(g.weights, orc.reciprocal(g.xadj, g.adj))
    return orc.propagate(g.xadj, g.adj, orc.hash_table(g.xadj, g.adj), thr, X, nthreads=4)[0]


def memoized(imx, g, r=16, seed=0):
    table = imx.build_hash_table(g)
    randoms = imx.SimulationRandoms(r, master_seed=seed)
    labels = imx.propagate(g, table, randoms)
    sizes, gains = imx.component_sizes_and_gains(labels, randoms.num_scored)
    return labels, sizes, gains, randoms.num_scored


# ---------------------------------------------------------------------------
# propagation (reference tests/test_propagation.py)
# ---------------------------------------------------------------------------

def test_weight_one_floods_min_label_everywhere(gpu, orc):
    g = weighted_er(gpu, 80, 5, "const:1.0")
    randoms = gpu.SimulationRandoms(16, 0)
    labels = gpu.propagate(g, gpu.build_hash_table(g), randoms)
    want = oracle_labels(orc, g, randoms)[:, 0]
    assert np.array_equal(labels, np.repeat(want[:, None], randoms.padded, axis=1))


def test_weight_zero_keeps_identity_labels(gpu):
    g = weighted_er(gpu, 80, 5, "const:0.0")
    randoms = gpu.SimulationRandoms(16, 0)
    labels, stats = gpu.propagate(g, gpu.build_hash_table(g), randoms, return_stats=True)
    assert np.array_equal(labels, np.repeat(np.arange(80, dtype=np.int32)[:, None], randoms.padded, axis=1))
    assert stats.sweeps == 1


def test_edgeless_graph_is_identity(gpu):
    g = gpu.Graph.from_edges(5, [])
    randoms = gpu.SimulationRandoms(16, 0)
    labels = gpu.propagate(g, gpu.build_hash_table(g), randoms)
    assert np.array_equal(labels, np.repeat(np.arange(5, dtype=np.int32)[:, None], randoms.padded, axis=1))


def test_path_with_middle_edge_dead(gpu):
    g = make_graph(gpu, [(0, 1), (1, 2)], weights=[1.0, 0.0])
    randoms = gpu.SimulationRandoms(16, 0)
    labels = gpu.propagate(g, gpu.build_hash_table(g), randoms)
    assert (labels[0] == 0).all() and (labels[1] == 0).all()
    assert (labels[2] == 2).all()


@pytest.mark.parametrize("scheme", ["const:0.15", "uniform:0.05,0.6", "normal:0.3,0.2", "wc"])
def test_partition_matches_oracle_lane_for_lane(gpu, orc, scheme):
    g = weighted_er(gpu, 150, 6, scheme, graph_seed=3, weight_seed=5)
    randoms = gpu.SimulationRandoms(24, master_seed=7)
    labels = gpu.propagate(g, gpu.build_hash_table(g), randoms)
    assert np.array_equal(labels, oracle_labels(orc, g, randoms))


def test_thread_counts_do_not_change_labels(gpu):
    g = weighted_er(gpu, 200, 8, "wc", graph_seed=9)
    table = gpu.build_hash_table(g)
    randoms = gpu.SimulationRandoms(32, master_seed=4)
    assert np.array_equal(gpu.propagate(g, table, randoms, n_threads=1),
                          gpu.propagate(g, table, randoms, n_threads=4))


def test_propagate_rejects_bad_widths(gpu):
    g = make_graph(gpu, [(0, 1)])
    table = gpu.build_hash_table(g)
    randoms = gpu.SimulationRandoms(16, 0)
    for bad in (12, 24, 0):
        with pytest.raises(ValueError):
            gpu.propagate(g, table, randoms, num_simulations=bad)


def test_stats_trace_invariants(gpu):
    g = weighted_er(gpu, 120, 6, "const:0.3", graph_seed=6)
    randoms = gpu.SimulationRandoms(16, master_seed=1)
    labels, stats = gpu.propagate(g, gpu.build_hash_table(g), randoms, return_stats=True)
    assert stats.sweeps == len(stats.modes) == len(stats.changed_pairs)
    assert stats.changed_pairs[-1] == 0
    sums = stats.label_sums
    assert len(sums) == stats.sweeps
    assert all(a >= b for a, b in zip(sums, sums[1:]))
    assert sums[-1] == labels.sum()


def test_narrower_width_is_prefix_of_wider(gpu):
    g = weighted_er(gpu, 100, 5, "const:0.2", graph_seed=2)
    table = gpu.build_hash_table(g)
    randoms = gpu.SimulationRandoms(32, master_seed=5)
    full = gpu.propagate(g, table, randoms)
    part = gpu.propagate(g, table, randoms, num_simulations=16)
    assert np.array_equal(full[:, :16], part)


def test_custom_hash_table_is_used(gpu, orc):
    """propagate(g, table, ...) samples with the table it is given."""
    g = weighted_er(gpu, 120, 6, "const:0.3", graph_seed=1)
    randoms = gpu.SimulationRandoms(16, 3)
    h = gpu.build_hash_table(g).hashes.copy()
    rec = g.reciprocal_slots
    alt = (h ^ 0x5A5A5A5) & 0x7FFFFFFF
    alt = np.minimum(alt, alt[rec])                    # keep it direction-oblivious
    custom = gpu.EdgeHashTable(alt)
    got = gpu.propagate(g, custom, randoms)
    thr = orc.thresholds(g.weights, orc.reciprocal(g.xadj, g.adj))
    want = orc.propagate(g.xadj, g.adj, alt, thr, randoms.values, nthreads=2)[0]
    assert np.array_equal(got, want)
    # the graph's own table is restored afterwards
    assert np.array_equal(gpu.propagate(g, gpu.build_hash_table(g), randoms), oracle_labels(orc, g, randoms))


def test_lane_label_step_pushes_only_into_v(gpu):
    from paper_2008_03095_b200.propagation import lane_label_step
    g = make_graph(gpu, [(0, 1), (1, 2)], weights=1.0)
    table = gpu.build_hash_table(g)
    randoms = gpu.SimulationRandoms(8, 0)
    labels = np.repeat(np.arange(3, dtype=np.int32)[:, None], 8, axis=1)
    assert lane_label_step(g, 1, 2, 0, labels, table, randoms)
    assert (labels[2] == 1).all()
    assert (labels[0] == 0).all() and (labels[1] == 1).all()
    assert lane_label_step(g, 0, 1, 0, labels, table, randoms)
    assert (labels[1] == 0).all()
    assert not lane_label_step(g, 0, 1, 0, labels, table, randoms)


def test_lane_label_step_respects_membership_and_alignment(gpu):
    from paper_2008_03095_b200.propagation import lane_label_step
    g = make_graph(gpu, [(0, 1)], weights=0.0)
    table = gpu.build_hash_table(g)
    randoms = gpu.SimulationRandoms(16, 0)
    labels = np.repeat(np.arange(2, dtype=np.int32)[:, None], 16, axis=1)
    assert not lane_label_step(g, 0, 1, 0, labels, table, randoms)
    assert (labels[1] == 1).all()
    with pytest.raises(ValueError):
        lane_label_step(g, 0, 1, 5, labels, table, randoms)
    with pytest.raises(ValueError):
        lane_label_step(g, 0, 1, 16, labels, table, randoms)


def test_component_sizes_and_gains_by_hand(gpu):
    labels = np.array([[0, 0], [0, 1], [2, 0]], dtype=np.int32)
    sizes = gpu.component_sizes(labels)
    assert sizes[:, 0].tolist() == [2, 0, 1]
    assert sizes[:, 1].tolist() == [2, 1, 0]
    gains = gpu.initial_marginal_gains(labels, sizes)
    assert gains.tolist() == [4, 3, 3]
    fs, fg = gpu.component_sizes_and_gains(labels)
    assert np.array_equal(fs, sizes) and np.array_equal(fg, gains)


def test_fused_pass_matches_two_pass_with_padding(gpu):
    g = weighted_er(gpu, 90, 6, "const:0.25", graph_seed=8)
    randoms = gpu.SimulationRandoms(20, master_seed=3)     # pads 20 -> 24
    labels = gpu.propagate(g, gpu.build_hash_table(g), randoms)
    sizes = gpu.component_sizes(labels)
    gains = gpu.initial_marginal_gains(labels, sizes, randoms.num_scored)
    fsizes, fgains = gpu.component_sizes_and_gains(labels, randoms.num_scored)
    assert np.array_equal(fsizes, sizes) and np.array_equal(fgains, gains)
    assert fgains.dtype == np.int64
    assert not np.array_equal(fgains, gpu.initial_marginal_gains(labels, sizes))


def test_dump_and_load_labels_round_trip(gpu, tmp_path):
    from paper_2008_03095_b200.propagation import dump_labels, load_labels
    g = weighted_er(gpu, 40, 4, "uniform:0.1,0.9", graph_seed=4)
    labels = gpu.propagate(g, gpu.build_hash_table(g), gpu.SimulationRandoms(8, 6))
    dump_labels(labels, tmp_path / "labels.bin")
    back = load_labels(tmp_path / "labels.bin")
    assert back.dtype == np.int32 and np.array_equal(back, labels)


# ---------------------------------------------------------------------------
# selection (reference tests/test_selection.py)
# ---------------------------------------------------------------------------

def test_two_components_pick_one_seed_each(gpu):
    g = make_graph(gpu, [(0, 1), (1, 2), (0, 2), (3, 4)], weights=1.0)
    labels, sizes, gains, r = memoized(gpu, g, r=8)
    res = gpu.select_seeds(g, labels, sizes, gains, k=2, num_scored=r)
    assert res.seeds == [0, 3]
    assert res.sigma == (3 + 2) * r and res.spread == 5.0
    assert res.gains == [3 * r, 2 * r]


def test_second_seed_in_same_component_adds_nothing(gpu):
    g = make_graph(gpu, [(0, 1), (1, 2)], weights=1.0)
    labels, sizes, gains, r = memoized(gpu, g, r=8)
    res = gpu.select_seeds(g, labels, sizes, gains, k=3, num_scored=r)
    assert res.seeds == [0, 1, 2] and res.gains == [3 * r, 0, 0] and res.spread == 3.0


def test_ties_break_to_smaller_vertex_id(gpu):
    g = make_graph(gpu, [(0, 1), (2, 3)], weights=1.0)
    labels, sizes, gains, r = memoized(gpu, g, r=8)
    assert gpu.select_seeds(g, labels, sizes, gains, k=2, num_scored=r).seeds == [0, 2]


def test_k_validation(gpu):
    g = make_graph(gpu, [(0, 1)])
    labels, sizes, gains, r = memoized(gpu, g)
    with pytest.raises(gpu.ConstraintError):
        gpu.select_seeds(g, labels, sizes, gains, k=0)
    with pytest.raises(gpu.ConstraintError, match="exceeds"):
        gpu.select_seeds(g, labels, sizes, gains, k=3)
    with pytest.raises(gpu.ConstraintError):
        gpu.run_fused(g, 3, num_simulations=8)


def test_commit_seed_owns_labels_and_banks_gain(gpu):
    g = make_graph(gpu, [(0, 1), (1, 2)], weights=1.0)
    labels, sizes, gains, r = memoized(gpu, g, r=8)
    state = gpu.SeedState.empty(g.n, r)
    first = gpu.marginal_gain(1, labels, sizes, state)
    assert first == 3 * r
    gpu.commit_seed(1, first, labels, state)
    assert state.seeds == [1] and state.sigma == 3 * r
    assert gpu.marginal_gain(0, labels, sizes, state) == 0
    assert gpu.recompute_sigma(labels, state) == state.sigma
    assert all(s == {0} for s in state.seed_label_sets())


def test_commit_seed_rejects_double_commit(gpu):
    g = make_graph(gpu, [(0, 1)], weights=1.0)
    labels, sizes, gains, r = memoized(gpu, g, r=8)
    state = gpu.SeedState.empty(g.n, r)
    gpu.commit_seed(0, gpu.marginal_gain(0, labels, sizes, state), labels, state)
    with pytest.raises(AssertionError):
        gpu.commit_seed(0, 0, labels, state)


def test_sigma_matches_independent_recount(gpu):
    g = weighted_er(gpu, 120, 6, "uniform:0.05,0.5", graph_seed=3, weight_seed=1)
    labels, sizes, gains, r = memoized(gpu, g, r=32, seed=2)
    res = gpu.select_seeds(g, labels, sizes, gains, k=8, num_scored=r)
    assert gpu.recompute_sigma(labels, res.state) == res.sigma == sum(res.gains)


def test_trace_lazy_evaluation_is_sound(gpu):
    g = weighted_er(gpu, 150, 7, "const:0.12", graph_seed=5)
    labels, sizes, gains, r = memoized(gpu, g, r=32, seed=4)
    res = gpu.select_seeds(g, labels, sizes, gains, k=10, num_scored=r)
    commits = [t for t in res.trace if t.committed]
    assert len(res.seeds) == len(commits) == 10
    for t in res.trace:
        assert t.fresh_gain <= t.stale_gain
        if t.committed:
            assert t.fresh_gain == t.stale_gain
    cg = [t.fresh_gain for t in commits]
    assert cg == sorted(cg, reverse=True) and cg == res.gains


def test_spread_se_matches_manual_computation(gpu):
    g = weighted_er(gpu, 60, 5, "const:0.3", graph_seed=7)
    randoms = gpu.SimulationRandoms(24, master_seed=6)
    labels = gpu.propagate(g, gpu.build_hash_table(g), randoms)
    sizes, gains = gpu.component_sizes_and_gains(labels, randoms.num_scored)
    res = gpu.select_seeds(g, labels, sizes, gains, k=4, num_scored=randoms.num_scored)
    sets = res.state.seed_label_sets()
    per_sim = np.array([sum(int(sizes[l, s]) for l in sets[s]) for s in range(randoms.num_scored)])
    assert per_sim.sum() == res.sigma
    want = per_sim.std(ddof=1) / np.sqrt(randoms.num_scored)
    assert res.spread_se(labels, sizes) == pytest.approx(want)


def test_spread_se_single_simulation_is_zero(gpu):
    g = make_graph(gpu, [(0, 1)], weights=1.0)
    labels = gpu.propagate(g, gpu.build_hash_table(g), gpu.SimulationRandoms(8, 0))
    sizes, gains = gpu.component_sizes_and_gains(labels, 1)
    res = gpu.select_seeds(g, labels, sizes, gains, k=1, num_scored=1)
    assert res.spread_se(labels, sizes) == 0.0


def test_write_trace_csv(gpu, tmp_path):
    g = weighted_er(gpu, 40, 4, "const:0.25", graph_seed=1)
    labels, sizes, gains, r = memoized(gpu, g, r=16, seed=3)
    res = gpu.select_seeds(g, labels, sizes, gains, k=3, num_scored=r)
    gpu.write_trace_csv(res.trace, tmp_path / "trace.csv")
    rows = list(csv.reader(open(tmp_path / "trace.csv", newline="")))
    assert rows[0] == ["vertex", "stale_gain", "fresh_gain", "committed", "seeds_before"]
    assert len(rows) == len(res.trace) + 1
    for row, rec in zip(rows[1:], res.trace):
        assert row == [str(rec.vertex), str(rec.stale_gain), str(rec.fresh_gain),
                       str(int(rec.committed)), str(rec.seeds_before)]


# ---------------------------------------------------------------------------
# pipeline (reference tests/test_pipeline.py)
# ---------------------------------------------------------------------------

def test_run_fused_composes_the_phases(gpu):
    g = weighted_er(gpu, 100, 6, "const:0.15", graph_seed=1, weight_seed=1)
    run = gpu.run_fused(g, 5, num_simulations=48, master_seed=7)
    labels = gpu.propagate(g, run.table, run.randoms)
    assert np.array_equal(run.labels, labels)
    sizes, gains = gpu.component_sizes_and_gains(labels, 48)
    assert np.array_equal(run.sizes, sizes)
    manual = gpu.select_seeds(g, labels, sizes, gains, 5, num_scored=48)
    assert run.seeds == manual.seeds and run.spread == manual.spread
    assert run.selection.sigma == manual.sigma
    assert run.spread_se == manual.spread_se(labels, sizes)


def test_run_fused_timings_and_id_mapping(gpu):
    # as_graph([(40, 41), (41, 42), (7, 8)]) compacts ids by first appearance
    g = gpu.Graph.from_edges(5, [(0, 1), (1, 2), (3, 4)], 1.0, orig_ids=[40, 41, 42, 7, 8])
    run = gpu.run_fused(g, 2, num_simulations=16, master_seed=0)
    assert set(run.timings) == {"hash", "propagate", "memoize", "select", "total"}
    assert all(v >= 0 for v in run.timings.values())
    assert run.timings["total"] >= run.timings["propagate"]
    assert run.original_seed_ids() == [40, 7] and run.seeds == [0, 3]


def test_run_fused_scores_only_requested_simulations(gpu):
    g = weighted_er(gpu, 60, 5, "const:0.2", graph_seed=2)
    run = gpu.run_fused(g, 3, num_simulations=20, master_seed=1)
    assert run.randoms.num_scored == 20 and run.selection.num_scored == 20
    assert run.labels.shape == (60, 24)


# ---------------------------------------------------------------------------
# hashing on the device (reference tests/test_hashing.py)
# ---------------------------------------------------------------------------

def test_pair_digest_reference_vectors_on_device(gpu):
    from paper_2008_03095_b200.hashing import _murmur3_pair_array
    for lo, hi, expected in [(0, 1, 0x3AD85688), (3, 7, 0x2C37C8F7), (123, 456, 0x33BE5BF3)]:
        assert gpu.murmur3_32(struct.pack("<II", lo, hi), 0) == expected
        got = _murmur3_pair_array(np.array([lo], np.uint32), np.array([hi], np.uint32))
        assert int(got[0]) == expected


def test_pair_array_matches_scalar_unmasked(gpu):
    from paper_2008_03095_b200.hashing import _murmur3_pair_array
    rng = np.random.default_rng(11)
    lo = rng.integers(0, 1 << 32, size=400, dtype=np.uint32)
    hi = rng.integers(0, 1 << 32, size=400, dtype=np.uint32)
    want = np.array([gpu.murmur3_32(struct.pack("<II", int(a), int(b)), 0) for a, b in zip(lo, hi)],
                    dtype=np.uint32)
    got = _murmur3_pair_array(lo, hi)
    assert got.dtype == np.uint32 and np.array_equal(got, want)


def test_hash_table_is_direction_oblivious_and_masked(gpu):
    g = weighted_er(gpu, 300, 6, "const:1.0", graph_seed=2)
    table = gpu.build_hash_table(g)
    h = table.hashes
    assert h.dtype == np.int32 and h.shape == (g.m,)
    assert (h >= 0).all() and (h <= gpu.H_MAX).all() and table.h_max == gpu.H_MAX
    assert np.array_equal(h, h[g.reciprocal_slots])


def test_hash_table_values_from_min_max_pair(gpu):
    g = gpu.Graph.from_edges(3, [(0, 1), (1, 2)])
    h = gpu.build_hash_table(g).hashes
    for u, v in [(0, 1), (1, 2)]:
        want = gpu.murmur3_32(struct.pack("<II", u, v), 0) & gpu.H_MAX
        assert int(h[g.slot(u, v)]) == want and int(h[g.slot(v, u)]) == want


def test_slot_thresholds_symmetrize_and_uniform(gpu):
    g = weighted_er(gpu, 60, 4, "const:1.0", graph_seed=1)
    w = np.random.default_rng(0).uniform(0.1, 0.9, size=g.m)
    g2 = g.with_weights(w)
    thr = gpu.slot_thresholds(g2, symmetrize=True)
    assert np.array_equal(thr, thr[g2.reciprocal_slots])
    assert (thr >= gpu.slot_thresholds(g2, symmetrize=False)).all()
    assert (gpu.slot_thresholds(g.with_weights(np.full(g.m, 0.25))) == gpu.threshold(0.25)).all()


def test_membership_rate_tracks_probability(gpu):
    g = weighted_er(gpu, 400, 8, "const:1.0", graph_seed=5)
    h = gpu.build_hash_table(g).hashes
    randoms = gpu.SimulationRandoms(512, master_seed=9)
    cells = np.bitwise_xor.outer(h, randoms.values)
    for p in (0.1, 0.5, 0.9):
        assert abs((cells < gpu.threshold(p)).mean() - p) < 0.02


def test_lane_membership_matches_scalar_rule(gpu):
    g = weighted_er(gpu, 120, 6, "const:1.0", graph_seed=8)
    table = gpu.build_hash_table(g)
    randoms = gpu.SimulationRandoms(24, master_seed=3)
    t = gpu.threshold(0.37)
    for slot in (0, 5, g.m - 1):
        for r0 in range(0, randoms.padded, gpu.LANE_WIDTH):
            mask = gpu.lane_membership(slot, r0, 0.37, table, randoms)
            for b in range(gpu.LANE_WIDTH):
                assert bool(mask >> b & 1) == ((int(randoms.values[r0 + b]) ^ int(table.hashes[slot])) < t)


def test_from_edges_validation_messages(gpu):
    with pytest.raises(ValueError, match="outside 0..n-1"):
        gpu.Graph.from_edges(3, [(0, 3)])
    with pytest.raises(ValueError, match="self-loops"):
        gpu.Graph.from_edges(3, [(1, 1)])
    with pytest.raises(ValueError, match="duplicate"):
        gpu.Graph.from_edges(3, [(0, 1), (1, 0)])
    with pytest.raises(gpu.ConstraintError):
        gpu.Graph.from_edges(-1, [])


# ---------------------------------------------------------------------------
# acceptance criteria (reference tests/test_acceptance.py)
# ---------------------------------------------------------------------------

def test_criterion_1_partition_oracle_equivalence(gpu, orc):
    widths = [8, 32, 64]
    rng = np.random.default_rng(2024)
    for i in range(60):
        n = int(np.exp(rng.uniform(np.log(4), np.log(1000))))
        deg = float(rng.uniform(1.0, min(8.0, n - 1)))
        g = weighted_er(gpu, n, deg, SCHEMES[i % 4], graph_seed=i, weight_seed=1000 + i)
        randoms = gpu.SimulationRandoms(widths[i % 3], master_seed=i)
        labels = gpu.propagate(g, gpu.build_hash_table(g), randoms)
        assert np.array_equal(labels, oracle_labels(orc, g, randoms)), f"instance {i}"


def test_criterion_2_greedy_reference_equivalence(gpu, orc):
    for i in range(40):
        rng = np.random.default_rng(3000 + i)
        n = int(rng.integers(3, 13))
        deg = float(rng.uniform(1.0, min(4.0, n - 1)))
        g = weighted_er(gpu, n, deg, SCHEMES[i % 4], graph_seed=i, weight_seed=i)
        k = int(rng.integers(1, n + 1))
        r = int(rng.choice([8, 16, 32]))
        run = gpu.run_fused(g, k, num_simulations=r, master_seed=i)
        want = orc.run_fused(g.xadj, g.adj, g.weights, k, r, i, nthreads=1)
        assert run.seeds == want["seeds"].tolist(), f"instance {i}"
        assert np.array_equal(run.selection.trace.array, want["trace"])


def test_criterion_5_fused_equals_oracle_on_er50k(gpu, orc):
    from paper_2008_03095_b200.generators import er_edges
    g = gpu.apply_weights(gpu.Graph.from_edges(50_000, er_edges(50_000, 200_000, 1)),
                          gpu.parse_weight_scheme("const:0.01"))
    run = gpu.run_fused(g, 10, num_simulations=256, master_seed=7)
    want = orc.run_fused(g.xadj, g.adj, g.weights, 10, 256, 7)
    assert run.seeds == want["seeds"].tolist()
    assert run.selection.sigma == want["sigma"]
    assert np.array_equal(run.labels, want["labels"])


def test_criterion_6_direction_obliviousness(gpu):
    for seed, scheme in enumerate(SCHEMES):
        g = weighted_er(gpu, 300, 6, scheme, graph_seed=seed, weight_seed=seed)
        table = gpu.build_hash_table(g)
        assert np.array_equal(table.hashes, table.hashes[g.reciprocal_slots])
        thr = gpu.slot_thresholds(g)
        assert np.array_equal(thr, thr[g.reciprocal_slots])


def test_criterion_6_sigma_consistency(gpu, orc):
    g = weighted_er(gpu, 150, 6, "uniform:0.05,0.6", graph_seed=31, weight_seed=3)
    randoms = gpu.SimulationRandoms(24, master_seed=9)
    labels = gpu.propagate(g, gpu.build_hash_table(g), randoms)
    sizes, gains = gpu.component_sizes_and_gains(labels, randoms.num_scored)
    res = gpu.select_seeds(g, labels, sizes, gains, 8, randoms.num_scored)
    assert gpu.recompute_sigma(labels, res.state) == res.sigma == sum(res.gains)
    # independent union count over the same worlds (labels of the seeds' components)
    cols = np.arange(randoms.num_scored)
    union = sum(int(np.isin(labels[:, r], labels[res.seeds, r]).sum()) for r in cols)
    assert union == res.sigma


def test_criterion_6_label_monotonicity(gpu):
    for seed, scheme in enumerate(SCHEMES):
        g = weighted_er(gpu, 400, 7, scheme, graph_seed=20 + seed, weight_seed=seed)
        _, stats = gpu.propagate(g, gpu.build_hash_table(g), gpu.SimulationRandoms(32, seed),
                                 return_stats=True)
        assert all(a >= b for a, b in zip(stats.label_sums, stats.label_sums[1:]))
        assert stats.changed_pairs[-1] == 0


def test_criterion_6_determinism_of_seeded_runs(gpu):
    g = weighted_er(gpu, 250, 6, "wc", graph_seed=50)
    a = gpu.run_fused(g, 6, num_simulations=64, master_seed=3)
    b = gpu.run_fused(g, 6, num_simulations=64, master_seed=3)
    assert a.seeds == b.seeds and a.selection.sigma == b.selection.sigma
    assert np.array_equal(a.labels, b.labels)
    assert np.array_equal(a.selection.trace.array, b.selection.trace.array)


@pytest.mark.parametrize("mode", [None, "enum", "dense"])
def test_caller_table_with_bit31_hashes_propagates_exactly(gpu, orc, mode, monkeypatch):
    # a caller-built EdgeHashTable may hold negative words: (X ^ h) is then
    # negative and always below thr (hashing.py:141-150); the device must not
    # use interval enumeration for such a table
    if mode:
        monkeypatch.setenv("IMX_HOOK", mode)
    g = weighted_er(gpu, 400, 6, "uniform:0.02,0.3", graph_seed=3, weight_seed=4)
    h = gpu.build_hash_table(g).hashes.copy()
    h[h % 7 == 0] |= np.int32(-2**31)          # reciprocal slots keep equal values
    table = gpu.EdgeHashTable(h)
    randoms = gpu.SimulationRandoms(40, master_seed=6)
    labels = gpu.propagate(g, table, randoms)
    thr = orc.thresholds(g.weights, orc.reciprocal(g.xadj, g.adj))
    want = orc.propagate(g.xadj, g.adj, h, thr, randoms.values, nthreads=4)[0]
    assert np.array_equal(labels, want)
