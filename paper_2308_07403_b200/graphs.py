"""The input contract of the hot path: a dense directed weight matrix.

Mirrors the reference's data model (pkg/src/rdist/graphs.py:20-116) so its
callers can pass the same objects: ``weights[i][j]`` is the weight of the edge
j -> i, ``+inf`` means no edge, and the diagonal is all ``+inf``. Graph
generators and edge-list file I/O of the reference are out of scope
(SURVEY.md 2.1 row 4); only what the path consumes lives here.

Any object with ``n_vertices``, ``weights`` and ``kind`` (whose ``.value`` is
"unweighted" / "integer" / "real") is accepted by the compute entry points,
so reference ``rdist.Graph`` instances work unchanged.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from pathlib import Path

import numpy as np


class GraphKind(Enum):
    """Weight class of a graph (graphs.py:20-23)."""

    UNWEIGHTED = "unweighted"
    INTEGER_WEIGHTED = "integer"
    REAL_WEIGHTED = "real"


def kind_value(g) -> str:
    """The kind string of our Graph or a duck-typed reference Graph."""
    k = g.kind
    return k.value if isinstance(k, Enum) else str(k)


@dataclass(frozen=True)
class Graph:
    """Immutable dense weighted digraph (graphs.py:26-68).

    Validation follows the reference: square float64 weights, all-inf
    diagonal, finite weights strictly positive, exactly 1.0 for unweighted and
    integral for integer-weighted graphs; the array is made read-only.
    """

    n_vertices: int
    weights: np.ndarray
    kind: GraphKind

    def __post_init__(self) -> None:
        w = np.asarray(self.weights, dtype=np.float64)
        object.__setattr__(self, "weights", w)
        n = self.n_vertices
        if n < 1:
            raise ValueError(f"n_vertices must be >= 1, got {n}")
        if w.shape != (n, n):
            raise ValueError(f"weights must be {n}x{n}, got {w.shape}")
        if not np.isinf(np.diagonal(w)).all():
            raise ValueError("diagonal entries must be +inf (no self-loops)")
        if np.isnan(w).any():
            raise ValueError("finite edge weights must be strictly positive")
        fin = w[np.isfinite(w)]
        if fin.size:
            if (fin <= 0).any():
                raise ValueError("finite edge weights must be strictly positive")
            if self.kind is GraphKind.UNWEIGHTED and (fin != 1.0).any():
                raise ValueError("unweighted graphs require all edge weights == 1.0")
            if self.kind is GraphKind.INTEGER_WEIGHTED and (fin != np.floor(fin)).any():
                raise ValueError("integer-weighted graphs require integral edge weights")
        w.setflags(write=False)

    def successors(self, i: int) -> np.ndarray:
        """Out-neighbours of vertex ``i`` in ascending order (graphs.py:61-63)."""
        return np.nonzero(np.isfinite(self.weights[:, i]))[0]

    @property
    def num_edges(self) -> int:
        return int(np.count_nonzero(np.isfinite(self.weights)))


@dataclass(frozen=True)
class EdgeList:
    """(from, to, weight) triples and the vertex count (graphs.py:71-76)."""

    vertex_count: int
    edges: tuple[tuple[int, int, float], ...]


def _weight_valid(kind: GraphKind, w: float) -> bool:
    if not (math.isfinite(w) and w > 0):
        return False
    if kind is GraphKind.UNWEIGHTED:
        return w == 1.0
    if kind is GraphKind.INTEGER_WEIGHTED:
        return float(w).is_integer()
    return True


def graph_from_edge_list(edges: EdgeList, kind: GraphKind) -> Graph:
    """Dense Graph from (from, to, weight) triples (graphs.py:89-111).

    ValueError on out-of-range vertices, self-loops, duplicate arcs or a
    weight the kind does not allow; the matrix stores ``w[to, from]``.
    """
    n = edges.vertex_count
    if n < 1:
        raise ValueError("vertex_count must be >= 1")
    w = np.full((n, n), np.inf)
    seen: set[tuple[int, int]] = set()
    for src, dst, weight in edges.edges:
        if not (0 <= src < n and 0 <= dst < n):
            raise ValueError(f"edge ({src}, {dst}) out of range for {n} vertices")
        if src == dst:
            raise ValueError(f"self-loop at vertex {src}")
        key = (src, dst)
        if key in seen:
            raise ValueError(f"duplicate edge ({src}, {dst})")
        if not _weight_valid(kind, weight):
            raise ValueError(f"weight {weight} invalid for kind {kind.value}")
        seen.add(key)
        w[dst, src] = weight
    return Graph(n, w, kind)


def adjacency_indicator(g) -> np.ndarray:
    """0/1 float64 matrix of the edge pattern (graphs.py:114-116)."""
    return np.isfinite(np.asarray(g.weights)).astype(np.float64)


# ---- wire formats either side of the path (graphs.py:284-329, cli.py:204-210)
def edge_list_from_graph(g) -> EdgeList:
    """(from, to, weight) triples of a Graph, sorted (graphs.py:284-290)."""
    w = np.asarray(g.weights)
    dst, src = np.nonzero(np.isfinite(w))
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    return EdgeList(int(g.n_vertices), tuple((int(s), int(d), float(w[d, s])) for s, d in zip(src, dst)))


def write_edge_list(edges: EdgeList, path) -> None:
    """``V <n>`` header, then one ``from to weight`` row per edge, weights with
    17 significant digits (graphs.py:293-297)."""
    rows = "".join(f"{s} {d} {w:.17g}\n" for s, d, w in edges.edges)
    Path(path).write_text(f"V {edges.vertex_count}\n" + rows, encoding="utf-8")


def read_edge_list(path) -> EdgeList:
    """Parse the edge-list format: ``#`` comments and blank lines ignored, the
    first entry must be ``V <vertex_count>`` (graphs.py:300-319)."""
    vertex_count = None
    triples: list[tuple[int, int, float]] = []
    for lineno, raw in enumerate(Path(path).read_text(encoding="utf-8").splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        parts = line.split()
        if vertex_count is None:
            if len(parts) != 2 or parts[0] != "V":
                raise ValueError(f"{path}:{lineno}: expected header 'V <vertex_count>'")
            vertex_count = int(parts[1])
            continue
        if len(parts) != 3:
            raise ValueError(f"{path}:{lineno}: expected 'from to weight'")
        triples.append((int(parts[0]), int(parts[1]), float(parts[2])))
    if vertex_count is None:
        raise ValueError(f"{path}: missing 'V <vertex_count>' header")
    return EdgeList(vertex_count, tuple(triples))


def infer_kind(edges: EdgeList) -> GraphKind:
    """Unweighted if every weight is 1, integer-weighted if all integral, else real (graphs.py:322-329)."""
    ws = np.array([w for _, _, w in edges.edges], dtype=np.float64)
    if np.all(ws == 1.0):
        return GraphKind.UNWEIGHTED
    if np.all(ws == np.floor(ws)):
        return GraphKind.INTEGER_WEIGHTED
    return GraphKind.REAL_WEIGHTED


def write_distance_csv(d, path) -> None:
    """One CSV row per distance row, ``inf`` for unreachable, 12 significant
    digits (the CLI's distance output, cli.py:204-210)."""
    d = np.asarray(d, dtype=np.float64)
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        for row in d:
            fh.write(",".join("inf" if np.isinf(v) else f"{v:.12g}" for v in row))
            fh.write("\n")
