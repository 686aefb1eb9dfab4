"""Shared fixtures: golden vectors, device detection, the gpu marker."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and libinfuser_b200.so")
    config.addinivalue_line("markers", "slow: long-running")
    config.addinivalue_line("markers", "scale: full BASELINE-config parity (minutes on the GPU box)")


def golden_names(prefix: str = "") -> list[str]:
    """Pipeline fixtures by default; evaluation / file-format / estimator ones
    under "eval_", "cdf_", "io_", "est_"."""
    names = sorted(p.stem for p in GOLDEN.glob(f"{prefix}*.npz"))
    if not prefix:
        names = [n for n in names if not n.startswith(("eval_", "cdf_", "io_", "est_"))]
    return names


def golden_graph(z: dict):
    """(xadj, adj, weights) of an evaluation fixture; config graphs are
    rebuilt from this repo's host generator (weights of the config scheme)."""
    if "cfg" in z:
        import oracle
        from paper_2008_03095_b200 import configs
        c = configs.CONFIGS[str(z["cfg"])]
        xadj, adj, _ = oracle.csr_from_edges(c.n, configs.edges(str(z["cfg"])))
        w = np.full(len(adj), float(c.weights.split(":")[1]))
        return xadj, adj, w
    return z["xadj"], z["adj"], z["weights"]


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def has_gpu() -> bool:
    try:
        from paper_2008_03095_b200 import _lib
        return _lib.load().imx_device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.fail("GPU test needs an sm_100 device and the built libinfuser_b200.so")
    import paper_2008_03095_b200 as imx
    return imx


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle
