"""B200-native Synchronised Louvain Method: the reference synclouvain's hot path
(local-move sweep, corrections, aggregation, modularity) on hand-written sm_100a CUDA.

Public surface mirrors the reference's (synclouvain/__init__.py:54-98) for the path:
``Graph.from_edges`` -> ``run(graph, RunConfig)`` -> ``RunResult`` plus the phase functions.
"""

from .detector import (Hierarchy, RunConfig, RunResult, RunStats, find_assignment,
                       maximal_correction, positive_correction, run)
from .forest import AssignmentForest, extract_components, reverse_assignment
from .graph import (Graph, GraphFormatError, NeighborUnion, Strengths, aggregate,
                    canonicalize_labels, compose_labels, strengths)
from .quality import CommunityAggregates, community_aggregates, gain_switch, local_gains, score
from .rng import uniform01

__all__ = [
    "AssignmentForest", "CommunityAggregates", "Graph", "GraphFormatError", "Hierarchy",
    "NeighborUnion", "RunConfig", "RunResult", "RunStats", "Strengths", "aggregate",
    "canonicalize_labels", "community_aggregates", "compose_labels", "extract_components",
    "find_assignment", "gain_switch", "local_gains", "maximal_correction",
    "positive_correction", "reverse_assignment", "run", "score", "strengths", "uniform01",
]
