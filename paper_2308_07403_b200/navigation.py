"""Greedy shortest-path pursuit on a distance estimate.

Mirrors ``greedy_descent`` / ``PathResult`` of pkg/src/rdist/navigation.py
(:19-24, :35-74). The per-step choice — the successor k of the current
vertex j minimising W[k][j] + dist[goal][k], lowest index on ties, stopping on
+inf — is computed on the GPU as a next-hop row (kernel K6) for the goal; the
walk is then a pointer chase over that row. ``next_hop_table`` evaluates the
same step for many goals at once (the config-4 table). The accuracy metrics
of the reference module are outside the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as _d
from . import _lib as L


@dataclass(frozen=True)
class PathResult:
    vertices: list[int]
    length: float
    reached: bool
    steps_taken: int


def _dist_rows_device(dist, rows: np.ndarray) -> torch.Tensor:
    dev = L.device()
    if isinstance(dist, torch.Tensor):
        d = dist.to(device=dev, dtype=torch.float64)
        return d[torch.as_tensor(rows, device=dev, dtype=torch.long)].contiguous()
    host = np.ascontiguousarray(np.asarray(dist, dtype=np.float64)[rows])
    return torch.from_numpy(host).to(dev)


def next_hop_rows(g, dist, targets) -> np.ndarray:
    """next[r][j] for goal targets[r] (int32, -1 = the walk stops at j)."""
    t = np.asarray(targets, dtype=np.int64).reshape(-1)
    n = g.n_vertices
    if t.size and (t.min() < 0 or t.max() >= n):
        raise ValueError(f"targets out of range for {n} vertices")
    w = _d.graph_weights(g)
    rows = _dist_rows_device(dist, t)
    tgt = torch.from_numpy(t.astype(np.int32)).to(w.device)
    return _d.next_hop(w, rows, tgt).cpu().numpy()


def next_hop_table(g, dist, targets=None, *, device_out: bool = False):
    """Next-hop table: row r is the greedy step toward ``targets[r]`` (default
    all vertices) from every vertex; entries are successors or -1."""
    n = g.n_vertices
    t = np.arange(n) if targets is None else np.asarray(targets, dtype=np.int64).reshape(-1)
    w = _d.graph_weights(g)
    if isinstance(dist, torch.Tensor) and targets is None:
        rows = dist.to(device=w.device, dtype=torch.float64).contiguous()
    else:
        rows = _dist_rows_device(dist, t)
    tgt = torch.from_numpy(t.astype(np.int32)).to(w.device)
    out = _d.next_hop(w, rows, tgt)
    return out if device_out else out.cpu().numpy()


def greedy_descent(g, dist: np.ndarray, start: int, goal: int, max_steps: int | None = None) -> PathResult:
    """Walk from start toward goal, always stepping to the successor k that
    minimises ``W[k][current] + dist[goal][k]`` (lowest index on ties); stops
    at the goal, after ``max_steps`` (default 4n), or when no successor has a
    finite score (navigation.py:35-74)."""
    n = g.n_vertices
    if not (0 <= start < n and 0 <= goal < n):
        raise ValueError(f"start/goal out of range for {n} vertices")
    if max_steps is None:
        max_steps = 4 * n
    path = [int(start)]
    length = 0.0
    current = int(start)
    steps = 0
    if current != goal and steps < max_steps:
        nxt = next_hop_rows(g, dist, [goal])[0]
        weights = np.asarray(g.weights)
        while current != goal and steps < max_steps:
            k = int(nxt[current])
            if k < 0:
                break
            length += float(weights[k, current])
            current = k
            path.append(current)
            steps += 1
    return PathResult(path, length, current == goal, steps)
