"""B200-native drop-in for the R-distance hot path of arXiv 2308.07403.

Same entry points, signatures, result types, exceptions and constants as the
reference package ``rdist`` for the path it accelerates:
``build_x``, ``resolvent``, ``r_distance``, ``rounded_r_distance``,
``lu_invert``, ``power_iteration`` / ``spectral_radius``, ``critical_gain``,
``precision_floor``, ``gamma_bounds``, ``suggest_gamma``, ``greedy_descent``;
plus the batched / table forms the B200 path adds
(``rounded_r_distance_batch``, ``next_hop_table``) and the distributed
inversion (``paper_2308_07403_b200.distributed``).

As in the reference (pkg/src/rdist/__init__.py:52-68) the re-exported
function ``resolvent`` shadows the submodule attribute of the same name.
"""

from .graphs import (
    EdgeList,
    Graph,
    GraphKind,
    adjacency_indicator,
    edge_list_from_graph,
    graph_from_edge_list,
    infer_kind,
    read_edge_list,
    write_distance_csv,
    write_edge_list,
)
from .linalg import (
    PIVOT_RTOL,
    PowerIterationResult,
    SingularMatrixError,
    lu_invert,
    mat_mul,
    power_iteration,
    spectral_radius,
)
from .navigation import AccuracyReport, PathResult, accuracy_report, greedy_descent, next_hop_table
from .resolvent import (
    DELTA_MIN,
    NEGATIVE_ENTRY_TOL,
    GammaBounds,
    HealthFlags,
    InfeasibleGammaError,
    ResolventResult,
    ResolventSingularError,
    build_x,
    communicability,
    critical_gain,
    gamma_bounds,
    precision_floor,
    r_distance,
    r_distance_device,
    resolvent,
    rounded_r_distance,
    suggest_gamma,
)
from .batch import (
    UNREACHABLE,
    UNREACHABLE_D8,
    bits_from_edge_list,
    decode_d8,
    rounded_r_distance_batch,
    rounded_r_distance_batch_device,
)
from ._lib import NativeUnavailableError, load_library
from .oracles import bfs_apsp, bfs_apsp_device, dijkstra_apsp, floyd_warshall, graph_diameter
from .navigation import global_accuracy, local_accuracy  # noqa: E402  (device K6/K9, .sweep)
from .sweep import SweepRecord, sweep_gamma_graph, sweep_point

__version__ = "0.1.0"

__all__ = [
    "DELTA_MIN",
    "NEGATIVE_ENTRY_TOL",
    "PIVOT_RTOL",
    "UNREACHABLE",
    "UNREACHABLE_D8",
    "bits_from_edge_list",
    "edge_list_from_graph",
    "infer_kind",
    "read_edge_list",
    "write_distance_csv",
    "write_edge_list",
    "bfs_apsp",
    "bfs_apsp_device",
    "dijkstra_apsp",
    "floyd_warshall",
    "graph_diameter",
    "AccuracyReport",
    "SweepRecord",
    "accuracy_report",
    "mat_mul",
    "global_accuracy",
    "local_accuracy",
    "sweep_gamma_graph",
    "sweep_point",
    "decode_d8",
    "EdgeList",
    "GammaBounds",
    "Graph",
    "GraphKind",
    "HealthFlags",
    "InfeasibleGammaError",
    "NativeUnavailableError",
    "PathResult",
    "PowerIterationResult",
    "ResolventResult",
    "ResolventSingularError",
    "SingularMatrixError",
    "adjacency_indicator",
    "build_x",
    "communicability",
    "critical_gain",
    "gamma_bounds",
    "graph_from_edge_list",
    "greedy_descent",
    "load_library",
    "lu_invert",
    "next_hop_table",
    "power_iteration",
    "precision_floor",
    "r_distance",
    "r_distance_device",
    "resolvent",
    "rounded_r_distance",
    "rounded_r_distance_batch",
    "rounded_r_distance_batch_device",
    "spectral_radius",
    "suggest_gamma",
]
