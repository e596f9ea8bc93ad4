"""Gamma sweep on the GPU.

The reference's accuracy harness — ``_sweep_point`` / ``sweep_gamma``
(pkg/src/rdist/experiments.py:138-211) over ``global_accuracy`` and
``local_accuracy`` (pkg/src/rdist/navigation.py:77-134) — evaluates, for one
graph and many gains, the rounded R-distance against the exact hop distances
and the greedy first step against the true shortest-path first steps. Here
every piece stays on the device:

* exact distances: K8 all-source BFS (:mod:`.oracles`), computed once per graph;
* per gamma: K1 -> K2 -> K3 through :func:`.resolvent.resolvent` (health
  flags with the reachable mask, as the reference passes it) and one K3 pass
  writing R and ceil(R);
* global accuracy: K9 count of ceil(R) == exact over finite off-diagonal pairs;
* local accuracy: K6 on the zero-weight pattern gives the estimate's chosen
  successor for every (goal, node) — the same first-minimum rule as the
  reference's ``argmin`` — and K9 checks it against the exact minimum over
  the successors (K6 on the exact distances, computed once per graph).

Results match the reference function by function on the same inputs
(tests/test_gpu_sweep.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as _d
from . import _lib as L
from .oracles import bfs_apsp_device
from .resolvent import ResolventSingularError, gamma_bounds, resolvent


@dataclass(frozen=True)
class SweepRecord:
    """One row of a gamma sweep (experiments.py:50-60)."""

    graph_family: str
    n_vertices: int
    gamma: float
    global_fraction: float
    local_fraction: float
    negative_entries: bool
    underflow_zeros: int
    gamma_over_critical: float
    precision_floor: float


def _dev(x) -> torch.Tensor:
    return _d.as_device_matrix(x)[0]


def _ratio(counts: torch.Tensor) -> float:
    ev, hit = (int(v) for v in counts.cpu().tolist())
    return float("nan") if ev == 0 else hit / ev


def global_accuracy(estimate, exact) -> float:
    """Fraction of ordered pairs (i != j, exact finite) with estimate == exact
    (navigation.py:77-88); NaN when nothing is evaluable. Host or device inputs."""
    est, ex = _dev(estimate), _dev(exact)
    if est.shape != ex.shape:
        raise ValueError(f"shape mismatch: {tuple(est.shape)} vs {tuple(ex.shape)}")
    n = ex.shape[0]
    counts = torch.zeros(2, dtype=torch.int64, device=ex.device)
    L.check(L.lib().rdb_global_accuracy(est.data_ptr(), est.stride(0), ex.data_ptr(), ex.stride(0), n,
                                        counts.data_ptr(), L.stream_handle()), "rdb_global_accuracy")
    return _ratio(counts)


class _GraphState:
    """Per-graph device state shared by every gamma of a sweep."""

    def __init__(self, g, exact=None):
        self.g = g
        self.n = n = g.n_vertices
        self.w = _d.graph_weights(g)
        # the estimate-only step (navigation.py:119-122) is K6 with every
        # finite weight replaced by 0: 0 + x == x exactly
        self.w0 = torch.where(torch.isfinite(self.w), torch.zeros_like(self.w), self.w)
        self.nnz = _d.count_edges(self.w0)
        self.exact = bfs_apsp_device(g) if exact is None else _dev(exact)
        self.targets = torch.arange(n, dtype=torch.int32, device=self.w.device)
        self.next_exact = _d.next_hop(self.w0, self.exact, self.targets, self.nnz)
        self.work = torch.empty(max(n, 1), dtype=torch.uint8, device=self.w.device)

    def local(self, est: torch.Tensor, atol: float) -> float:
        next_est = _d.next_hop(self.w0, est, self.targets, self.nnz)
        counts = torch.zeros(2, dtype=torch.int64, device=est.device)
        L.check(
            L.lib().rdb_local_accuracy(self.w.data_ptr(), self.w.stride(0), next_est.data_ptr(),
                                       self.next_exact.data_ptr(), next_est.stride(0), est.data_ptr(),
                                       est.stride(0), self.exact.data_ptr(), self.exact.stride(0),
                                       self.targets.data_ptr(), self.n, self.n, float(atol), self.work.data_ptr(),
                                       counts.data_ptr(), L.stream_handle()),
            "rdb_local_accuracy",
        )
        return _ratio(counts)


def local_accuracy(g, estimate, exact, atol: float = 0.0) -> float:
    """Fraction of (goal, node) pairs whose estimate-predicted successor is one
    of the truly closest successors (navigation.py:91-134)."""
    est, ex = _dev(estimate), _dev(exact)
    if est.shape != ex.shape:
        raise ValueError(f"shape mismatch: {tuple(est.shape)} vs {tuple(ex.shape)}")
    return _GraphState(g, ex).local(est.contiguous(), atol)


def _reachable_mask(exact: torch.Tensor) -> torch.Tensor:
    n = exact.shape[0]
    m = torch.isfinite(exact)
    m.fill_diagonal_(False)
    return m.to(torch.uint8)


def sweep_point(family: str, g, exact, reachable, gamma: float, gc: float, floor: float,
                state: _GraphState | None = None) -> SweepRecord:
    """One gamma of the sweep, the reference's ``_sweep_point`` (experiments.py:138-167)."""
    st = state if state is not None else _GraphState(g, exact)
    over = gamma / gc if math.isfinite(gc) else 0.0
    try:
        res = resolvent(g, gamma, reachable=reachable)
    except ResolventSingularError:
        return SweepRecord(family, g.n_vertices, gamma, 0.0, 0.0, True, 0, over, floor)
    y = res.device_y()
    raw, rounded = _d.log_ceil(y, st.n, gamma, want_r=True, want_dceil=True)
    return SweepRecord(
        graph_family=family,
        n_vertices=g.n_vertices,
        gamma=gamma,
        global_fraction=global_accuracy(rounded, st.exact),
        local_fraction=st.local(raw, 0.0),
        negative_entries=res.health.negative_entries,
        underflow_zeros=res.health.underflow_zeros or 0,
        gamma_over_critical=over,
        precision_floor=floor,
    )


def default_gamma_grid(bounds, per_decade: int = 32, decades_below_floor: float = 2.0) -> np.ndarray:
    """Log grid from below the precision floor to twice the critical gain (experiments.py:124-135)."""
    lo = max(bounds.precision_floor_for_dmax * 10.0**-decades_below_floor, 1e-300)
    gc = min(bounds.critical_gain, 1.0)
    hi = min(2.0 * gc, 0.99)
    if hi <= lo:
        hi = min(0.99, lo * 10.0)
    n_points = max(2, round(math.log10(hi / lo) * per_decade) + 1)
    return np.geomspace(lo, hi, n_points)


def sweep_gamma_graph(g, gammas=None, family: str = "", per_decade: int = 32) -> list[SweepRecord]:
    """The inner loop of ``sweep_gamma`` (experiments.py:170-211) for one
    graph: exact distances once (K8), then every gamma on the device."""
    st = _GraphState(g)
    finite = st.exact[torch.isfinite(st.exact)]
    d_max = max(int(finite.max().item()) if finite.numel() else 0, 1)
    bounds = gamma_bounds(g, d_max)
    grid = np.asarray(gammas, dtype=np.float64) if gammas is not None else default_gamma_grid(bounds, per_decade)
    reach = _reachable_mask(st.exact)
    out = [sweep_point(family, g, st.exact, reach, float(gm), bounds.critical_gain, bounds.precision_floor_for_dmax,
                       state=st) for gm in grid]
    out.sort(key=lambda r: (r.graph_family, r.n_vertices, r.gamma))
    return out
