"""Bit-exact parity at the BASELINE configs' full scale (GPU).

north_star: bit-exact seeds and scores versus the CPU oracle on all 5
configs.  Each test runs the device ``run_fused`` on a config graph and
checks, over EVERY lane (oracle/scale_check.py):

* the labels and sizes of every lane chunk against the oracle's per-lane
  union-find (pinned to the reference's fixtures in test_oracle_golden.py);
* the initial gains, seeds, seed gains, sigma, the full CELF dequeue trace
  and spread_se against the reference's CELF heap run on the exact
  fresh-gain table;
* for the largest configs, a window of lanes at each end of the matrix
  against the dense min-label restatement (oracle.propagate).

These are the code paths that only switch on at scale: 8/16-wave compress
grids, lane-tiled compression with the fused memo (C5), 16 blocks/SM
enumeration above 1e8 live pairs (C4), CELF rounds refreshing millions of
vertices (C4), the late weight upload (> 4M slots), gains above 2^32 (C5).
The graph is generated on the device (configs.build), and its CSR is
compared with the host restatement for the configs whose host build is
cheap.
"""

import gc

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.scale]

_GRAPHS = {}


def config_graph(gpu, cfg):
    """Device-generated config graph, cached for the module (C4: ~3 GB)."""
    from paper_2008_03095_b200 import configs
    if cfg not in _GRAPHS:
        _GRAPHS.clear()
        gc.collect()
        _GRAPHS[cfg] = configs.build(cfg)
    return _GRAPHS[cfg]


@pytest.mark.parametrize("cfg", ["c1", "c2", "c2p1", "c3", "c5"])
def test_config_csr_matches_host_restatement(gpu, orc, cfg):
    """Device generator + CSR build == numpy generator + the oracle's CSR
    (Graph.from_edges, graph.py:124-155) and thresholds (hashing.py:153-165)."""
    from paper_2008_03095_b200 import configs
    g = config_graph(gpu, cfg)
    c = configs.CONFIGS[cfg]
    xadj, adj, _ = orc.csr_from_edges(c.n, configs.edges(cfg))
    assert np.array_equal(g.xadj, xadj) and np.array_equal(g.adj, adj)
    thr = orc.thresholds(np.asarray(g.weights), orc.reciprocal(xadj, adj))
    assert np.array_equal(gpu.slot_thresholds(g), thr)


@pytest.mark.parametrize("cfg,R,dense", [
    ("c2", None, 0), ("c2p1", None, 0), ("c3", None, 16),
    ("c4", 64, 0), ("c4", None, 8),
    ("c5", 64, 0), ("c5", None, 8),
])
def test_run_fused_matches_oracle_at_config_scale(gpu, orc, cfg, R, dense):
    """run_fused(g, K, R) on the config graph: every lane's labels and sizes,
    the gains, seeds, seed gains, sigma, trace and spread_se equal the
    oracle's (R=None: the config's full R; R=64: the reduced-R variant)."""
    from oracle.scale_check import check_fused_run
    from paper_2008_03095_b200 import configs
    c = configs.CONFIGS[cfg]
    g = config_graph(gpu, cfg)
    R = R or c.R
    run = gpu.run_fused(g, c.K, num_simulations=R, master_seed=0)
    rep = check_fused_run(run, g, c.K, R, 0, dense_window=dense)
    del run
    gc.collect()
    print(cfg, R, rep)
    assert rep["ok"], rep
