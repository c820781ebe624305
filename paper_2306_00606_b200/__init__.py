"""B200-native Expected Force engine -- drop-in for the efgraph EF path.

Public surface mirrors efgraph/__init__.py:3-20 for the hot path: graph
construction (Graph, RmatParams, build_graph, generate_rmat, cluster_count)
and Expected Force (EFResult, cluster_degree, ef, ef_cluster_centric,
ef_vertex_centric, entropy_from_histogram, write_ef_csv), plus key_nodes
(device top-k) and the ranking consumers of analysis.py (ef_bins,
ef_rank_ascending, immunization_windows).  The compute runs in libefg.so (sm_100a CUDA behind the C ABI
of include/efg.h); importing this package does not touch the GPU.
"""
from .graph import (
    DEFAULT_RMAT_PROBS,
    Graph,
    RmatParams,
    build_graph,
    cluster_count,
    generate_rmat,
)
from .expected_force import (
    FLAG_NO_CLUSTERS,
    FLAG_OK,
    FLAG_ZERO_DEGREE_CLUSTERS,
    EFResult,
    cluster_degree,
    ef,
    ef_cluster_centric,
    ef_vertex_centric,
    entropy_from_histogram,
    key_nodes,
    write_ef_csv,
)
from .io import load_edge_list, write_edge_list
from .ranking import EFBin, ef_bins, ef_rank_ascending, immunization_windows
from ._native import EFGDeviceError, set_device

__version__ = "0.1.0"
