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


def edges(name: str) -> np.ndarray:
    c = CONFIGS[name]
    if name == "c1":
        return gen.chung_lu_edges(c.n, 31_000, 2.5, c.seed)
    if name in ("c2", "c2p1"):
        return gen.chung_lu_edges(c.n, 174_000, 2.2, c.seed)
    if name == "c3":
        return gen.rmat_edges(18, c.seed, m=1_230_000)
    if name == "c4":
        return gen.rmat_edges(22, c.seed, edge_factor=16)
    if name == "c5":
        return gen.er_edges(c.n, 5_000_000, c.seed)
    raise KeyError(name)


def build(name: str, edge_list: np.ndarray | None = None):
    """Device-built Graph with the config's weights applied."""
    from .graph import Graph
    from .weights import apply_weights, parse_weight_scheme
    c = CONFIGS[name]
    e = edges(name) if edge_list is None else edge_list
    g = Graph.from_edges(c.n, e)
    return apply_weights(g, parse_weight_scheme(c.weights), rng_seed=c.seed)
