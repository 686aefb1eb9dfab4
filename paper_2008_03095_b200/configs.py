"""The five BASELINE.json configurations as seeded synthetic workloads.

graph_seed = weight_seed = config number, master_seed = 0.
``edges(name)`` is host-only (numpy); ``build(name)`` builds the device CSR
and applies the weight scheme.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import generators as gen

__all__ = ["Config", "CONFIGS", "edges", "build"]


@dataclass(frozen=True)
class Config:
    name: str
    description: str
    n: int
    weights: str          # parse_weight_scheme text
    R: int
    K: int
    seed: int


CONFIGS = {
    "c1": Config("c1", "Chung-Lu gamma=2.5 n=15000 m=31000 p=0.01 R=128 K=20",
                 15_000, "const:0.01", 128, 20, 1),
    "c2": Config("c2", "Chung-Lu gamma=2.2 n=37000 m=174000 p=0.01 R=1024 K=50",
                 37_000, "const:0.01", 1024, 50, 2),
    "c2p1": Config("c2p1", "Chung-Lu gamma=2.2 n=37000 m=174000 p=0.1 R=1024 K=50",
                   37_000, "const:0.1", 1024, 50, 2),
    "c3": Config("c3", "R-MAT(.57,.19,.19,.05) scale 18 m=1230000 p~N(0.05,0.025) R=2048 K=50",
                 1 << 18, "normal:0.05,0.025", 2048, 50, 3),
    "c4": Config("c4", "R-MAT(.57,.19,.19,.05) scale 22 edge factor 16 p=0.005 R=1024 K=100",
                 1 << 22, "const:0.005", 1024, 100, 4),
    "c5": Config("c5", "Erdos-Renyi G(n=1000000, m=5000000) p=0.05 R=8192 K=50",
                 1_000_000, "const:0.05", 8192, 50, 5),
}


_RMAT = (0.57, 0.19, 0.19, 0.05)


def _spec(name: str):
    """(kind, n, m, draws, probs, cdf) of a config's generator."""
    c = CONFIGS[name]
    if name == "c1":
        return gen.CHUNG_LU, c.n, 31_000, 0, None, gen.chung_lu_cdf(c.n, 2.5)
    if name in ("c2", "c2p1"):
        return gen.CHUNG_LU, c.n, 174_000, 0, None, gen.chung_lu_cdf(c.n, 2.2)
    if name == "c3":
        return gen.RMAT, c.n, 1_230_000, 0, _RMAT, None
    if name == "c4":
        return gen.RMAT, c.n, 0, 16 * c.n, _RMAT, None
    if name == "c5":
        return gen.ER, c.n, 5_000_000, 0, None, None
    raise KeyError(name)


def edges(name: str) -> np.ndarray:
    """Host (numpy) edge list -- identical to the device generator's."""
    kind, n, m, draws, probs, cdf = _spec(name)
    return gen.edges(kind, n, m, CONFIGS[name].seed, draws, probs, cdf)


def build(name: str, edge_list: np.ndarray | None = None):
    """Graph with the config's weights applied; generated on the device
    unless an edge list is given."""
    from .graph import Graph
    from .weights import apply_weights, parse_weight_scheme
    c = CONFIGS[name]
    if edge_list is None:
        kind, n, m, draws, probs, cdf = _spec(name)
        g = gen.device_graph(kind, n, m, c.seed, draws, probs, cdf)
    else:
        g = Graph.from_edges(c.n, edge_list)
    return apply_weights(g, parse_weight_scheme(c.weights), rng_seed=c.seed)
