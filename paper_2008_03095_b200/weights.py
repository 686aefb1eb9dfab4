"""Diffusion-probability schemes (reference graph.py:162-266).

Host plumbing that prepares the per-slot weights the sampler thresholds are
derived from.  The draws must be the reference's: one numpy PCG64 draw per
undirected edge, taken in canonical-slot order (slots whose source is the
smaller endpoint) and written to both directions; weighted cascade is the
per-direction 1/deg(target).  The scheme names and the text syntax
('const:P', 'uniform:LO,HI', 'normal:MEAN,STD', 'wc', 'file') are the
reference's public surface.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._lib import ConstraintError
from .graph import Graph

__all__ = ["Constant", "UniformRange", "NormalClamped", "WeightedCascade", "FromFile",
           "parse_weight_scheme", "apply_weights"]


@dataclass(frozen=True)
class Constant:
    """Every edge gets probability p in both directions."""
    p: float


@dataclass(frozen=True)
class UniformRange:
    """One uniform draw in [lo, hi] per undirected edge."""
    lo: float
    hi: float


@dataclass(frozen=True)
class NormalClamped:
    """One N(mean, std) draw per undirected edge, clamped into [0, 1]."""
    mean: float
    std: float


@dataclass(frozen=True)
class WeightedCascade:
    """weight(u, v) = 1 / degree(v)."""


@dataclass(frozen=True)
class FromFile:
    """Keep the weights already stored on the graph."""


_SCHEMES = (Constant, UniformRange, NormalClamped, WeightedCascade, FromFile)


def _validate(scheme, exc):
    """Range checks shared by the parser (ValueError) and apply (ConstraintError)."""
    if isinstance(scheme, Constant) and not 0.0 <= scheme.p <= 1.0:
        raise exc(f"probability {scheme.p} outside [0, 1]")
    if isinstance(scheme, UniformRange) and not 0.0 <= scheme.lo <= scheme.hi <= 1.0:
        raise exc(f"range [{scheme.lo}, {scheme.hi}] invalid")
    if isinstance(scheme, NormalClamped) and (not 0.0 <= scheme.mean <= 1.0 or scheme.std < 0.0):
        raise exc(f"normal({scheme.mean}, {scheme.std}) parameters invalid")
    return scheme


def parse_weight_scheme(text):
    """'const:P' | 'uniform:LO,HI' | 'normal:MEAN,STD' | 'wc' | 'file' -> scheme
    (graph.py:195-227); scheme objects pass through unchanged."""
    if isinstance(text, _SCHEMES):
        return text
    name, _, args = str(text).partition(":")
    arity = {"const": (Constant, 1), "uniform": (UniformRange, 2),
             "normal": (NormalClamped, 2), "wc": (WeightedCascade, 0),
             "file": (FromFile, 0)}
    if name not in arity:
        raise ValueError(f"unknown weight scheme {text!r}")
    cls, count = arity[name]
    if count == 0:
        if args:
            raise ValueError(f"unknown weight scheme {text!r}")
        return cls()
    try:
        values = [float(a) for a in args.split(",")]
        if len(values) != count:
            raise ValueError(f"expected {count} parameter(s)")
        return _validate(cls(*values), ValueError)
    except ValueError as exc:
        raise ValueError(f"bad weight scheme {text!r}: {exc}") from None


def _per_edge(g: Graph, draws: np.ndarray) -> np.ndarray:
    canon = g.canonical_slots
    w = np.empty(g.m, dtype=np.float64)
    w[canon] = draws
    w[g.reciprocal_slots[canon]] = draws
    return w


def apply_weights(g: Graph, scheme, rng_seed: int = 0) -> Graph:
    """New Graph with per-slot weights from ``scheme`` (graph.py:230-266)."""
    if not isinstance(scheme, _SCHEMES):
        raise TypeError(f"unknown weight scheme {scheme!r}")
    _validate(scheme, ConstraintError)
    if isinstance(scheme, FromFile):
        return g.with_weights(g.weights)
    if isinstance(scheme, Constant):
        return g.with_weights(np.full(g.m, scheme.p, dtype=np.float64))
    if isinstance(scheme, WeightedCascade):
        return g.with_weights(1.0 / g.degrees[g.adj])
    rng = np.random.default_rng(rng_seed)
    count = len(g.canonical_slots)
    if isinstance(scheme, UniformRange):
        draws = rng.uniform(scheme.lo, scheme.hi, size=count)
    else:
        draws = np.clip(rng.normal(scheme.mean, scheme.std, size=count), 0.0, 1.0)
    return g.with_weights(_per_edge(g, draws))
