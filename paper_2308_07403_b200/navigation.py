"""Greedy shortest-path pursuit on a distance estimate.

Mirrors ``greedy_descent`` / ``PathResult`` of pkg/src/rdist/navigation.py
(:19-24, :35-74). The per-step choice — the successor k of the current
vertex j minimising W[k][j] + dist[goal][k], lowest index on ties, stopping on
+inf — is computed on the GPU as a next-hop row (kernel K6) for the goal; the
walk is then a pointer chase over that row. ``next_hop_table`` evaluates the
same step for many goals at once (the config-4 table; ``next_hop_table_shard``
gives one rank its block of target rows). The reference module's accuracy
metrics (navigation.py:77-153: global_accuracy, local_accuracy,
accuracy_report / AccuracyReport) run on the device (K6 + K9, :mod:`.sweep`).
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


@dataclass(frozen=True)
class AccuracyReport:
    """navigation.py:27-32."""

    global_fraction: float
    local_fraction: float
    pairs_evaluated: int
    pairs_excluded_unreachable: int


def global_accuracy(estimate, exact) -> float:
    """Fraction of off-diagonal exact-finite pairs where estimate == exact
    (navigation.py:77-88), counted on the device (K9)."""
    from .sweep import global_accuracy as _g

    return _g(estimate, exact)


def local_accuracy(g, estimate, exact, atol: float = 0.0) -> float:
    """Fraction of (goal, node) pairs whose estimate-predicted successor is a
    truly closest successor (navigation.py:91-134), on the device (K6 + K9)."""
    from .sweep import local_accuracy as _l

    return _l(g, estimate, exact, atol=atol)


def accuracy_report(g, global_estimate, local_estimate, exact, atol: float = 0.0) -> AccuracyReport:
    """Both metrics at once (navigation.py:137-153): the rounded estimate feeds
    the global metric, the raw one the local metric; pair counts from the
    exact distances."""
    ex = np.asarray(exact) if not isinstance(exact, torch.Tensor) else exact.detach().cpu().numpy()
    off = ~np.eye(ex.shape[0], dtype=bool)
    fin = np.isfinite(ex)
    return AccuracyReport(
        global_fraction=global_accuracy(global_estimate, exact),
        local_fraction=local_accuracy(g, local_estimate, exact, atol=atol),
        pairs_evaluated=int((off & fin).sum()),
        pairs_excluded_unreachable=int((off & ~fin).sum()),
    )


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


def shard_targets(n: int, rank: int, world: int) -> np.ndarray:
    """Contiguous block of target rows owned by ``rank`` of ``world`` (config 4
    sharded by target rows: W and dist replicated, no exchange)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return np.arange(lo, hi)


def next_hop_table_shard(g, dist, rank: int | None = None, world: int | None = None, *, device_out: bool = False):
    """This rank's rows of the next-hop table (targets ``shard_targets``); rank
    and world default to the initialised torch.distributed group (one process
    per GPU), else (0, 1). Returns (targets, table rows)."""
    if rank is None or world is None:
        import torch.distributed as dist_mod

        if dist_mod.is_available() and dist_mod.is_initialized():
            rank, world = dist_mod.get_rank(), dist_mod.get_world_size()
        else:
            rank, world = 0, 1
    t = shard_targets(g.n_vertices, rank, world)
    if t.size == 0:
        return t, np.empty((0, g.n_vertices), dtype=np.int32)
    return t, next_hop_table(g, dist, t, device_out=device_out)


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
