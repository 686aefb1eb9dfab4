"""Host restatement of the counter-based generators (CPU-only)."""

import numpy as np

from conftest import load_golden


def test_streams_are_prefix_stable_and_deterministic():
    from paper_2008_03095_b200 import generators as gen
    a = gen._candidates(gen.ER, 1000, 7, 0, 500)
    b = gen._candidates(gen.ER, 1000, 7, 0, 2000)
    assert np.array_equal(a, b[:500])
    assert np.array_equal(gen._candidates(gen.ER, 1000, 7, 100, 50), b[100:150])
    assert not np.array_equal(a, gen._candidates(gen.ER, 1000, 8, 0, 500))


def test_first_m_distinct_edges():
    from paper_2008_03095_b200 import generators as gen
    e = gen.edges(gen.ER, 200, 900, 3)
    assert e.shape == (900, 2)
    assert (e[:, 0] < e[:, 1]).all()
    assert len(np.unique(e[:, 0] * 200 + e[:, 1])) == 900
    # a larger m extends the same draw order
    e2 = gen.edges(gen.ER, 200, 950, 3)
    assert np.array_equal(e2[:900], e)


def test_rmat_skew_and_all_distinct_mode():
    from paper_2008_03095_b200 import generators as gen
    e = gen.edges(gen.RMAT, 1 << 10, 0, 5, draws=16 << 10, probs=(0.57, 0.19, 0.19, 0.05))
    deg = np.bincount(e.ravel(), minlength=1 << 10)
    assert deg[:16].mean() > 5 * deg.mean()          # hubs at low ids
    assert len(np.unique(e[:, 0] * 1024 + e[:, 1])) == len(e)


def test_bench_configs_match_golden_edges():
    from paper_2008_03095_b200 import configs
    for cfg in ("c1", "c2"):
        z = load_golden(f"cfg_{cfg}")
        assert np.array_equal(configs.edges(cfg), z["edges"].astype(np.int64))
