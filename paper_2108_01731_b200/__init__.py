"""B200-native LambdaCC best-move / contraction hot path (arXiv 2108.01731).

Public API mirrors the reference specification (``/root/reference/SPEC.md``):
objective (``cc_objective``, ``modularity_params``, ``modularity_value``,
``rescaled_weight``, ``move_delta``) and louvain-par (``ParOptions``,
``par_best_moves``, ``compute_frontier``, ``par_compress``, ``par_flatten``,
``parallel_cc``, ``per_vertex_best_target``).  All computation runs in the
sm_100a library ``_lib/liblcc_b200.so`` (C ABI: ``include/lcc_b200.h``).
"""
from ._lib import NativeLibraryError
from .graph import DeviceGraph, GraphError, build_graph, build_graph_arrays
from .objective import (Clustering, ClusteringParams, cc_objective, clustering_from_labels, modularity_params,
                        modularity_value, move_delta, rescaled_weight, singletons)
from .louvain_par import (CompressedLevel, Frontier, FrontierPolicy, MoveBuffer, ParOptions, RunStats, Schedule,
                          apply_moves, best_moves_round, compute_frontier, frontier_from_mask, par_best_moves, release_memory, par_compress,
                          par_flatten, parallel_cc, per_vertex_best_target)

__all__ = [
    "NativeLibraryError", "DeviceGraph", "GraphError", "build_graph", "build_graph_arrays", "Clustering", "ClusteringParams", "cc_objective",
    "clustering_from_labels", "modularity_params", "modularity_value", "move_delta", "rescaled_weight",
    "singletons", "CompressedLevel", "Frontier", "FrontierPolicy", "MoveBuffer", "ParOptions", "RunStats",
    "Schedule", "apply_moves", "best_moves_round", "compute_frontier", "frontier_from_mask", "par_best_moves", "release_memory",
    "par_compress", "par_flatten", "parallel_cc", "per_vertex_best_target",
]
