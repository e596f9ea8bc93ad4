"""Small graph builders for the tests (the reference's generators are outside
the hot path and not part of the package)."""

import numpy as np

from paper_2308_07403_b200 import EdgeList, Graph, GraphKind, graph_from_edge_list


def undirected(n, pairs):
    w = np.full((n, n), np.inf)
    for a, b in pairs:
        w[a, b] = w[b, a] = 1.0
    return Graph(n, w, GraphKind.UNWEIGHTED)


def grid(side):
    pairs = []
    for y in range(side):
        for x in range(side):
            i = y * side + x
            if x + 1 < side:
                pairs.append((i, i + 1))
            if y + 1 < side:
                pairs.append((i, i + side))
    return undirected(side * side, pairs)


def binary_tree(levels):
    n = 2**levels - 1
    return undirected(n, [(i, (i - 1) // 2) for i in range(1, n)])


def dense(n, p, seed):
    rng = np.random.default_rng(seed)
    present = rng.random((n, n)) < p
    np.fill_diagonal(present, False)
    return Graph(n, np.where(present, 1.0, np.inf), GraphKind.UNWEIGHTED)


def weighted(n, p, lo, hi, seed):
    rng = np.random.default_rng(seed)
    present = rng.random((n, n)) < p
    np.fill_diagonal(present, False)
    w = np.exp(rng.uniform(np.log(lo), np.log(hi), size=(n, n)))
    return Graph(n, np.where(present, w, np.inf), GraphKind.REAL_WEIGHTED)


def chain2():
    return graph_from_edge_list(EdgeList(2, ((0, 1, 1.0),)), GraphKind.UNWEIGHTED)


def ring3():
    return graph_from_edge_list(EdgeList(3, tuple((i, (i + 1) % 3, 1.0) for i in range(3))), GraphKind.UNWEIGHTED)


def empty(n):
    return graph_from_edge_list(EdgeList(n, ()), GraphKind.UNWEIGHTED)


def directed_path(n):
    return graph_from_edge_list(EdgeList(n, tuple((i, i + 1, 1.0) for i in range(n - 1))), GraphKind.UNWEIGHTED)


def u8_to_d(u8):
    d = u8.astype(np.float64)
    d[u8 == 255] = np.inf
    return d


def d_digest(d_u8) -> bytes:
    """Digest of a D in the compact byte form (uint8, 255 = +inf), as
    tests/golden/make_golden_full.py stores the reference's."""
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(d_u8, dtype=np.uint8).tobytes()).digest()[:16]


def int32_to_u8(d32):
    """int32 D (INT32_MAX = unreachable, all finite D <= 254) -> uint8 form."""
    fin = d32 != np.iinfo(np.int32).max
    assert (d32[fin] >= 0).all() and (d32[fin] <= 254).all()
    out = np.full(d32.shape, 255, np.uint8)
    out[fin] = d32[fin]
    return out


def f64_to_u8(d):
    fin = np.isfinite(d)
    out = np.full(d.shape, 255, np.uint8)
    out[fin] = d[fin].astype(np.uint8)
    return out
