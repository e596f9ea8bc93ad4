"""Exact distances on the GPU: the reference's ``bfs_apsp``
(pkg/src/rdist/oracles.py:22-41) as kernel K8 (csrc/bfs.cu) and its
``floyd_warshall`` (:44-50) as kernel K10 (csrc/floyd.cu, bit for bit the
same k-loop), which also serves ``dijkstra_apsp`` (:53-66): on positive
weights both are the shortest-path lengths (exactly equal on integer
weights; the reference's Dijkstra sums paths in another order, so on real
weights it matches to float tolerance, as the reference's own docstring says).

The reference advances all-source BFS frontiers with dense boolean matrix
products; K8 keeps the frontiers bit-packed by source and ORs, for every
vertex, the frontier rows of its in-neighbours (a sparse-row x bit-matrix
product per level), writing each distance once. Same output convention:
``d[i][j]`` = hops from j to i, 0 on the diagonal, +inf (or INT32_MAX for
int32 output) when unreachable. It is the exact side of the gamma sweep
(:mod:`.sweep`) and verifies D at sizes the CPU oracle cannot reach.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _device as _d
from . import _lib as L
from .graphs import kind_value


def pattern_bits(w: torch.Tensor) -> torch.Tensor:
    """Device bit-packed adjacency (n, ceil(n/32)) int32 of a device weight matrix."""
    n = w.shape[0]
    bits = torch.empty((n, (n + 31) // 32), dtype=torch.int32, device=w.device)
    L.check(L.lib().rdb_pattern_bits(w.data_ptr(), n, w.stride(0), bits.data_ptr(), L.stream_handle()),
            "rdb_pattern_bits")
    return bits


def bfs_apsp_bits(bits: torch.Tensor, n: int, dtype: torch.dtype = torch.float64) -> tuple[torch.Tensor, int]:
    """(distances, deepest level) from device bit-packed adjacency (rdb_build_m_bits row format)."""
    if dtype not in (torch.float64, torch.int32):
        raise ValueError("dtype must be torch.float64 or torch.int32")
    dev = bits.device
    dist = torch.empty((n, n), dtype=dtype, device=dev)
    work = torch.empty(L.lib().rdb_bfs_workspace_bytes(n), dtype=torch.uint8, device=dev)
    levels = ctypes.c_int64(0)
    d32 = dist.data_ptr() if dtype == torch.int32 else None
    d64 = dist.data_ptr() if dtype == torch.float64 else None
    L.check(L.lib().rdb_bfs_apsp(bits.data_ptr(), n, d32, d64, n, work.data_ptr(), ctypes.byref(levels),
                                 L.stream_handle()), "rdb_bfs_apsp")
    return dist, int(levels.value)


def bfs_apsp_device(g, dtype: torch.dtype = torch.float64) -> torch.Tensor:
    """As :func:`bfs_apsp`, result left on the device."""
    if kind_value(g) != "unweighted":
        raise ValueError(f"bfs_apsp requires an unweighted graph, got {kind_value(g)}")
    w = _d.graph_weights(g)
    return bfs_apsp_bits(pattern_bits(w), g.n_vertices, dtype)[0]


def bfs_apsp(g) -> np.ndarray:
    """Exact distances on an unweighted graph (oracles.py:22-41): float64,
    +inf when unreachable, zero diagonal."""
    return bfs_apsp_device(g).cpu().numpy()


def floyd_warshall_device(g) -> torch.Tensor:
    """Floyd-Warshall distances of a graph (any kind) on the device (K10)."""
    w = _d.graph_weights(g)
    n = g.n_vertices
    d = torch.empty((n, n), dtype=torch.float64, device=w.device)
    work = torch.empty(L.lib().rdb_floyd_workspace_bytes(n), dtype=torch.uint8, device=w.device)
    L.check(L.lib().rdb_floyd_warshall(w.data_ptr(), w.stride(0), n, d.data_ptr(), n, work.data_ptr(),
                                       L.stream_handle()), "rdb_floyd_warshall")
    return d


def floyd_warshall(g) -> np.ndarray:
    """Exact weighted distances (oracles.py:44-50): d[i][j] from j to i, +inf
    unreachable, zero diagonal; the reference's loop bit for bit."""
    return floyd_warshall_device(g).cpu().numpy()


def dijkstra_apsp(g) -> np.ndarray:
    """Exact weighted distances (oracles.py:53-66), computed by K10."""
    return floyd_warshall(g)


def graph_diameter(d: np.ndarray) -> float:
    """Largest finite entry of an exact distance matrix, 0 if none (oracles.py:110-113)."""
    d = np.asarray(d)
    finite = d[np.isfinite(d)]
    return float(finite.max()) if finite.size else 0.0
