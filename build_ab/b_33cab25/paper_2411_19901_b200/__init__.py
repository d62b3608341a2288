"""B200-native drop-in for the sketchlpa label-propagation hot path
(arXiv 2411.19901: nuMG8-LPA / nuBM-LPA).

Public names mirror sketchlpa/__init__.py:33-55 for the hot path:
LpaConfig, LpaResult, lpa_run, lpa_move, aux_memory_estimate, modularity,
community_stats, CommunityStats, Graph, build_graph.  The compute runs in
libslpa_b200.so (hand-written sm_100a CUDA) through a C ABI
(include/slpa.h); there is no CPU fallback.
"""

from .engine import Engine, default_engine, keep_threshold, rmat_thresholds
from .graph import Graph, GraphLoadError, build_graph, build_graph_arrays
from .graph_io import load_graph, validate_graph, write_edgelist, write_matrix_market
from .lpa import LpaConfig, LpaResult, aux_memory_estimate, lpa_move, lpa_run
from .metrics import CommunityStats, community_stats, modularity

__version__ = "0.1.0"

__all__ = [
    "CommunityStats",
    "Engine",
    "Graph",
    "GraphLoadError",
    "LpaConfig",
    "LpaResult",
    "aux_memory_estimate",
    "build_graph",
    "build_graph_arrays",
    "community_stats",
    "default_engine",
    "keep_threshold",
    "load_graph",
    "lpa_move",
    "lpa_run",
    "modularity",
    "rmat_thresholds",
    "validate_graph",
    "write_edgelist",
    "write_matrix_market",
]
