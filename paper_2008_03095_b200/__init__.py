"""paper_2008_03095_b200 -- B200-native hot path of InFuseR-MG (arxiv 2008.03095).

Drop-in for the reference ``infmax`` entry points of the fused path: hash-
sampled Independent-Cascade simulation over R implicit samples, per-sample
connected components (min vertex id labels), memoized component-size gains
and CELF seed selection -- all computed by the sm_100a kernels of
libinfuser_b200.so (include/infuser_b200.h).  There is no CPU fallback.
"""

from ._lib import ConstraintError, GraphFormatError, set_device
from .estimator import InfluenceMaximizer
from .evaluation import (KS_UNIFORM_BOUND, SamplingCdf, evaluate_seeds, sampling_cdf,
                         write_cdf_tsv)
from .graph import MAX_VERTICES, Graph
from .io import load_csr, load_edge_list, load_graph, save_csr, write_edge_list
from .hashing import (H_MAX, LANE_WIDTH, EdgeHashTable, SimulationRandoms, build_hash_table,
                      lane_membership, murmur3_32, sample_prob, slot_thresholds, threshold)
from .pipeline import FusedRun, run_fused
from .propagation import (PropagateStats, component_sizes, component_sizes_and_gains,
                          initial_marginal_gains, propagate)
from .selection import (SeedState, SelectionResult, TraceRecord, commit_seed, marginal_gain,
                        recompute_sigma, select_seeds, write_trace_csv)
from .weights import (Constant, FromFile, NormalClamped, UniformRange, WeightedCascade,
                      apply_weights, parse_weight_scheme)

__version__ = "0.1.0"

__all__ = [
    "InfluenceMaximizer", "load_csr", "load_edge_list", "load_graph", "save_csr", "write_edge_list",
    "KS_UNIFORM_BOUND", "SamplingCdf", "evaluate_seeds", "sampling_cdf", "write_cdf_tsv",
    "ConstraintError", "Constant", "EdgeHashTable", "FromFile", "FusedRun", "Graph",
    "GraphFormatError", "H_MAX", "LANE_WIDTH", "MAX_VERTICES", "NormalClamped",
    "PropagateStats", "SeedState", "SelectionResult", "SimulationRandoms", "TraceRecord",
    "UniformRange", "WeightedCascade", "apply_weights", "build_hash_table", "commit_seed",
    "component_sizes", "component_sizes_and_gains", "initial_marginal_gains",
    "lane_membership", "marginal_gain", "murmur3_32", "parse_weight_scheme", "propagate",
    "recompute_sigma", "run_fused", "sample_prob", "select_seeds", "set_device",
    "slot_thresholds", "threshold", "write_trace_csv",
]
