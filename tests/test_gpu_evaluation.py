"""evaluate_seeds / sampling_cdf on the device vs. the reference (GPU).

The golden fixtures hold the reference's own per-world counts, (mean, se)
and SamplingCdf fields (tests/golden/make_golden_eval.py); the device must
reproduce them exactly -- counts bit for bit, mean/se/ks/cdf as identical
float64.  Config-scale cases are checked against the pinned C oracle.
"""

import hashlib
import os

import numpy as np
import pytest

from conftest import golden_graph, golden_names, load_golden

pytestmark = pytest.mark.gpu

EVAL = golden_names("eval_")
CDF = golden_names("cdf_")


def _graph(imx, xadj, adj, w):
    return imx.Graph(np.asarray(xadj, np.int64), np.asarray(adj, np.int32), np.asarray(w, np.float64),
                     np.arange(len(xadj) - 1, dtype=np.int64))


def make_graph(imx, edges, n=None, weights=1.0):
    edges = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if n is None:
        n = int(edges.max()) + 1
    return imx.Graph.from_edges(n, edges, weights)


def weighted_er(imx, n, deg, scheme, graph_seed=0, weight_seed=0):
    from paper_2008_03095_b200.generators import er_edges
    g = imx.Graph.from_edges(n, er_edges(n, int(round(n * deg / 2)), graph_seed))
    return imx.apply_weights(g, imx.parse_weight_scheme(scheme), rng_seed=weight_seed)


@pytest.mark.parametrize("name", EVAL)
def test_evaluate_matches_reference(gpu, name):
    from paper_2008_03095_b200.evaluation import evaluate_counts
    z = load_golden(name)
    g = _graph(gpu, *golden_graph(z))
    counts = evaluate_counts(g, z["seeds"], int(z["r_eval"]), int(z["rng_seed"]))
    assert np.array_equal(counts, z["counts"])
    assert gpu.evaluate_seeds(g, z["seeds"], int(z["r_eval"]), int(z["rng_seed"])) == \
        (float(z["mean"]), float(z["se"]))


@pytest.mark.parametrize("worlds", ["64", "100", "4000"])
def test_evaluate_batches_split_chunks(gpu, worlds, monkeypatch):
    # worlds of one chunk split over several label-matrix batches
    from paper_2008_03095_b200.evaluation import evaluate_counts
    z = load_golden("eval_er1000")
    g = _graph(gpu, z["xadj"], z["adj"], z["weights"])
    monkeypatch.setenv("IMX_EVAL_WORLDS", worlds)
    counts = evaluate_counts(g, z["seeds"], int(z["r_eval"]), int(z["rng_seed"]))
    assert np.array_equal(counts, z["counts"])


@pytest.mark.parametrize("cfg,r_eval,k", [("c2", 8200, 50), ("c3", 700, 40)])
def test_evaluate_config_scale_vs_oracle(gpu, orc, cfg, r_eval, k):
    from paper_2008_03095_b200 import configs
    from paper_2008_03095_b200.evaluation import evaluate_counts
    g = configs.build(cfg)
    seeds = np.random.default_rng(k).choice(g.n, size=k, replace=False)
    counts = evaluate_counts(g, seeds, r_eval, 17)
    want = orc.evaluate_counts(g.xadj, g.adj, g.weights, seeds, r_eval, 17)
    assert np.array_equal(counts, want)


def test_evaluate_many_seeds_and_duplicates(gpu, orc):
    g = weighted_er(gpu, 3000, 6, "uniform:0.05,0.4", 2, 3)
    seeds = np.random.default_rng(0).integers(0, g.n, size=900)   # many duplicates
    from paper_2008_03095_b200.evaluation import evaluate_counts
    counts = evaluate_counts(g, seeds, 5000, 4)
    want = orc.evaluate_counts(g.xadj, g.adj, g.weights, seeds, 5000, 4)
    assert np.array_equal(counts, want)


# ---- ports of the reference's tests/test_evaluation.py:30-85 ---------------

def test_evaluate_is_deterministic_and_thread_invariant(gpu):
    g = weighted_er(gpu, 200, 6, "const:0.1", graph_seed=1)
    a = gpu.evaluate_seeds(g, [0, 5, 9], 10_000, rng_seed=3)
    b = gpu.evaluate_seeds(g, [0, 5, 9], 10_000, rng_seed=3)
    c = gpu.evaluate_seeds(g, [0, 5, 9], 10_000, rng_seed=3, n_threads=4)
    assert a == b == c
    assert a != gpu.evaluate_seeds(g, [0, 5, 9], 10_000, rng_seed=4)


def test_evaluate_exact_at_weight_extremes(gpu):
    g = make_graph(gpu, [(0, 1), (1, 2), (3, 4)], weights=1.0)
    assert gpu.evaluate_seeds(g, [0], 100) == (3.0, 0.0)
    assert gpu.evaluate_seeds(g, [0, 3], 100) == (5.0, 0.0)
    g0 = make_graph(gpu, [(0, 1), (1, 2)], weights=0.0)
    assert gpu.evaluate_seeds(g0, [1], 100) == (1.0, 0.0)


def test_evaluate_deduplicates_and_validates(gpu):
    g = make_graph(gpu, [(0, 1)], weights=1.0)
    assert gpu.evaluate_seeds(g, [0, 0, 1], 10) == (2.0, 0.0)
    with pytest.raises(ValueError):
        gpu.evaluate_seeds(g, [], 10)
    with pytest.raises(ValueError):
        gpu.evaluate_seeds(g, [4], 10)
    with pytest.raises(ValueError):
        gpu.evaluate_seeds(g, [0], 0)


def test_evaluate_single_world_has_zero_se(gpu):
    g = make_graph(gpu, [(0, 1)], weights=0.5)
    mean, se = gpu.evaluate_seeds(g, [0], 1)
    assert mean in (1.0, 2.0) and se == 0.0


def test_evaluate_edgeless_graph(gpu):
    g = gpu.Graph.from_edges(6, np.zeros((0, 2), np.int64))
    assert gpu.evaluate_seeds(g, [0, 2, 5], 300, rng_seed=1) == (3.0, 0.0)


# ---- sampling_cdf ------------------------------------------------------------

@pytest.mark.parametrize("name", CDF)
def test_sampling_cdf_matches_reference(gpu, name):
    z = load_golden(name)
    if "cfg" in z:
        from paper_2008_03095_b200 import configs
        g = configs.build(str(z["cfg"]))
        assert hashlib.sha256(g.adj.tobytes()).hexdigest() == str(z["adj_sha"])
    else:
        g = _graph(gpu, z["xadj"], z["adj"], np.ones(len(z["adj"])))
    table = gpu.build_hash_table(g)
    if bool(z["broken"]):
        table = gpu.EdgeHashTable(np.zeros(g.m, np.int32))
    randoms = gpu.SimulationRandoms(int(z["R"]), master_seed=int(z["master_seed"]))
    assert np.array_equal(randoms.values, z["X"])
    res = gpu.sampling_cdf(g, table, randoms, bins=int(z["bins"]))
    assert res.num_values == int(z["num_values"])
    assert res.ks_distance == float(z["ks"])
    assert np.array_equal(res.cdf, z["cdf"]) and np.array_equal(res.bin_uppers, z["bin_uppers"])
    # the graph samples with its own table again afterwards
    gpu.build_hash_table(g).bind(g)


def test_sampling_cdf_is_near_uniform_and_broken_is_not(gpu):
    from paper_2008_03095_b200.generators import er_edges
    g = gpu.Graph.from_edges(2000, er_edges(2000, 10_000, 4))
    randoms = gpu.SimulationRandoms(256, master_seed=0)
    res = gpu.sampling_cdf(g, gpu.build_hash_table(g), randoms)
    assert res.num_values == g.num_undirected_edges * 256
    assert res.uniform_ok and res.ks_distance < 0.01
    assert res.cdf[-1] == pytest.approx(1.0) and (np.diff(res.cdf) >= 0).all()
    bad = gpu.sampling_cdf(g, gpu.EdgeHashTable(np.zeros(g.m, np.int32)), randoms)
    assert not bad.uniform_ok


def test_sampling_cdf_ks_matches_manual(gpu, orc):
    from paper_2008_03095_b200.generators import er_edges
    g = gpu.Graph.from_edges(100, er_edges(100, 200, 1))
    table = gpu.build_hash_table(g)
    randoms = gpu.SimulationRandoms(8, master_seed=2)
    res = gpu.sampling_cdf(g, table, randoms, bins=50)
    canon = g.canonical_slots
    vals = np.sort((np.bitwise_xor.outer(table.hashes[canon], randoms.values) / (2**31 - 1)).ravel())
    k = len(vals)
    want = max((np.arange(1, k + 1) / k - vals).max(), (vals - np.arange(k) / k).max())
    assert res.ks_distance == want
    assert len(res.bin_uppers) == len(res.cdf) == 50


def test_sampling_cdf_validates_bins_and_writes_tsv(gpu, tmp_path):
    from paper_2008_03095_b200.generators import er_edges
    g = gpu.Graph.from_edges(50, er_edges(50, 100, 0))
    table = gpu.build_hash_table(g)
    randoms = gpu.SimulationRandoms(8, master_seed=0)
    with pytest.raises(ValueError):
        gpu.sampling_cdf(g, table, randoms, bins=5)
    res = gpu.sampling_cdf(g, table, randoms, bins=20)
    path = tmp_path / "cdf.tsv"
    gpu.write_cdf_tsv(res, path)
    rows = [line.split("\t") for line in path.read_text().splitlines()]
    assert len(rows) == 20 and float(rows[-1][0]) == 1.0
    assert float(rows[-1][1]) == pytest.approx(1.0)


@pytest.mark.parametrize("bins", [10, 100, 1000, 20000])
def test_sampling_cdf_histogram_rule_vs_numpy(gpu, orc, bins):
    # numpy's uniform-bin corrections, including the smem/global paths
    from paper_2008_03095_b200.generators import er_edges
    g = gpu.Graph.from_edges(3000, er_edges(3000, 12_000, 9))
    randoms = gpu.SimulationRandoms(96, master_seed=5)
    res = gpu.sampling_cdf(g, gpu.build_hash_table(g), randoms, bins=bins)
    up, cdf, ks, k = orc.sampling_cdf(g.xadj, g.adj, orc.hash_table(g.xadj, g.adj), randoms.values, 96, bins)
    assert res.num_values == k and res.ks_distance == ks and np.array_equal(res.cdf, cdf)


def test_sampling_cdf_edgeless_raises(gpu):
    g = gpu.Graph.from_edges(4, np.zeros((0, 2), np.int64))
    with pytest.raises(ValueError):
        gpu.sampling_cdf(g, gpu.build_hash_table(g), gpu.SimulationRandoms(8))
