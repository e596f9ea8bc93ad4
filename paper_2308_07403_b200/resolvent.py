"""Shortest-path distances from a single matrix inversion — the drop-in.

Mirrors pkg/src/rdist/resolvent.py (names, signatures, result types,
exceptions, constants). The pipeline X = gamma^W, M = 1 - X, Y = M^-1,
R = log Y / log gamma, D = ceil R runs as sm_100a kernels (K1 build-M, K2
Gauss-Jordan DMMA inversion, K3 log/ceil, K5 residual, K4 power iteration);
numpy arrays are only the host-side inputs and outputs. The resolvent result
keeps Y on the device, so r_distance / rounded_r_distance of it never move Y
through the host; ``ResolventResult.y`` materialises a host copy lazily.

The scalar gamma-window helpers (precision_floor, gamma_bounds,
suggest_gamma) are host arithmetic, as in the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as _d
from . import _lib as L
from .graphs import kind_value
from .linalg import PIVOT_RTOL, SingularMatrixError

# Smallest positive subnormal float64 (resolvent.py:24).
DELTA_MIN = math.ulp(0.0)

NEGATIVE_ENTRY_TOL = -1e-12  # resolvent.py:26


class ResolventSingularError(RuntimeError):
    """(1 - X) was singular to working precision (resolvent.py:29-38)."""

    def __init__(self, gamma: float):
        super().__init__(
            f"resolvent inapplicable at gamma={gamma:.6g}: (1 - X) is singular "
            "to working precision"
        )
        self.gamma = gamma


class InfeasibleGammaError(ValueError):
    """No gamma can satisfy both the precision floor and the critical gain."""


@dataclass(frozen=True)
class HealthFlags:
    """Numerical-health summary of one resolvent computation (resolvent.py:45-57)."""

    negative_entries: bool
    underflow_zeros: int | None
    inversion_residual: float


class _HostY:
    """Data descriptor behind ``ResolventResult.y``: the host array, copied
    from the device matrix on first access when the result came from
    :func:`resolvent` (which keeps Y on the GPU). Raising AttributeError on
    class access tells ``dataclass`` the field has no default."""

    def __get__(self, obj, owner=None):
        if obj is None:
            raise AttributeError("y")
        d = obj.__dict__
        if d.get("_y_host") is None and d.get("_y_dev") is not None:
            n = d["_n"]
            d["_y_host"] = d["_y_dev"][:n, :n].cpu().numpy().copy(order="C")
        return d.get("_y_host")

    def __set__(self, obj, value):  # reached only through object.__setattr__ (frozen)
        obj.__dict__["_y_host"] = value
        if value is not None:
            obj.__dict__["_n"] = np.asarray(value).shape[0]


@dataclass(frozen=True)
class ResolventResult:
    """(y, gamma, health) as the reference's frozen dataclass (resolvent.py:60-64):
    same fields, so ``dataclasses.fields/replace/asdict`` work for drop-in
    callers. A result made by :func:`resolvent` also holds Y on the device
    (``device_y()``); ``y`` is then copied to the host on first access."""

    y: np.ndarray = _HostY()
    gamma: float
    health: HealthFlags

    @classmethod
    def _on_device(cls, y_dev: torch.Tensor, n: int, gamma: float, health: HealthFlags) -> "ResolventResult":
        res = cls(None, gamma, health)
        object.__setattr__(res, "_y_dev", y_dev)
        object.__setattr__(res, "_n", n)
        return res

    def device_y(self) -> torch.Tensor:
        """Y on the CUDA device (an n x n view, possibly of a padded buffer)."""
        d = self.__dict__
        if d.get("_y_dev") is None:
            t = torch.from_numpy(np.ascontiguousarray(d["_y_host"], dtype=np.float64)).to(L.device())
            object.__setattr__(self, "_y_dev", t)
        n = d["_n"]
        return d["_y_dev"][:n, :n]

    def __repr__(self) -> str:
        return f"ResolventResult(n={self.__dict__.get('_n')}, gamma={self.gamma!r}, health={self.health!r})"


@dataclass(frozen=True)
class GammaBounds:
    """Feasibility window for gamma on a given graph (resolvent.py:67-87)."""

    critical_gain: float
    precision_floor_for_dmax: float
    d_max_used: int
    feasible: bool
    delta: float = DELTA_MIN

    @property
    def max_feasible_distance(self) -> float:
        """Largest d_max the float format supports below the critical gain."""
        if self.critical_gain >= 1.0:
            return math.inf
        return math.log(self.delta) / math.log(self.critical_gain)


def _check_gamma(gamma: float) -> None:
    if not 0 < gamma < 1:
        raise ValueError(f"gamma must be in (0, 1), got {gamma}")


def build_x(g, gamma: float) -> np.ndarray:
    """Entry-wise gamma**W with gamma**inf = 0 (resolvent.py:90-98), on the GPU."""
    _check_gamma(gamma)
    w = _d.graph_weights(g)
    x = _d.build_m(w, g.n_vertices, gamma, mode=L.RDB_BUILD_X)
    return x.cpu().numpy()


def resolvent(g, gamma: float, reachable: np.ndarray | None = None, with_residual: bool = True) -> ResolventResult:
    """Invert (1 - gamma**W) and report numerical health (resolvent.py:101-128).

    Raises ResolventSingularError (chained from SingularMatrixError) when a
    pivot falls below PIVOT_RTOL * max|M|.
    """
    _check_gamma(gamma)
    n = g.n_vertices
    w = _d.graph_weights(g)
    n_pad = L.pad_to_nb(n)
    m_pad = _d.build_m(w, n, gamma, n_pad)
    scale, nonfinite, nonz, _ = _d.matrix_stats(m_pad[:n, :n])
    m_keep = m_pad.clone() if with_residual else None
    try:
        if nonfinite:
            raise _d.InversionFailure(math.nan, scale)
        y_pad = _invert_m(m_pad, n, scale, nonz == 0, lambda: _d.build_m(w, n, gamma, n_pad))
    except _d.InversionFailure as exc:
        raise ResolventSingularError(gamma) from SingularMatrixError(str(exc))
    counters = torch.zeros(L.RDB_NCOUNTERS, dtype=torch.int64, device=y_pad.device)
    reach_dev = None
    if isinstance(reachable, torch.Tensor):  # device mask (the GPU sweep passes one)
        reach_dev = reachable.to(device=y_pad.device, dtype=torch.uint8).contiguous()
    elif reachable is not None:
        r = np.ascontiguousarray(np.asarray(reachable, dtype=bool)).view(np.uint8)
        reach_dev = torch.from_numpy(r).to(y_pad.device)
    _d.log_ceil(y_pad, n, gamma, reachable=reach_dev, counters=counters)
    cnt = counters.cpu().tolist()
    negative = cnt[L.RDB_CNT_NEGATIVE] > 0
    underflow = int(cnt[L.RDB_CNT_UNDERFLOW]) if reachable is not None else None
    residual = math.nan
    if with_residual:
        residual = _d.residual(m_keep, y_pad)
    return ResolventResult._on_device(y_pad, n, gamma, HealthFlags(negative, underflow, residual))


def _invert_m(m_pad: torch.Tensor, n: int, scale: float, z_matrix: bool, rebuild) -> torch.Tensor:
    """Inverse of the padded M: in place by the no-pivot DMMA kernel when its
    pivots certify a nonsingular M-matrix and pass the reference's rule, else
    (on a rebuilt M) by the partial-pivoting kernel, whose pivots then decide
    singularity exactly as LAPACK's getrf pivots do in linalg.py:32-38."""
    tol = PIVOT_RTOL * scale
    if scale == 0.0:
        raise _d.InversionFailure(0.0, scale)
    if z_matrix:
        rec = _d.invert_padded_nopivot(m_pad)
        if not (rec.flags & (L.RDB_PIV_NONPOS | L.RDB_PIV_NONFINITE)) and rec.min_pivot >= tol:
            return m_pad
        m_pad = rebuild()
    y = _d.invert(m_pad[:n, :n].contiguous(), scale, False, PIVOT_RTOL)
    return _d.pad_copy(y, m_pad.shape[0])


def _device_y_of(res) -> tuple[torch.Tensor, int]:
    if isinstance(res, ResolventResult):
        yd = res.device_y()
        return yd, yd.shape[0]
    y = np.ascontiguousarray(np.asarray(res.y, dtype=np.float64))
    t = torch.from_numpy(y).to(L.device())
    return t, y.shape[0]


def r_distance(res) -> np.ndarray:
    """log Y / log gamma entry-wise, +inf where Y <= 0, zero diagonal (resolvent.py:131-143)."""
    y, n = _device_y_of(res)
    r, _ = _d.log_ceil(y, n, res.gamma, want_r=True)
    return r.cpu().numpy()


def rounded_r_distance(res) -> np.ndarray:
    """ceil(r_distance(res)) without nudge (resolvent.py:146-153)."""
    y, n = _device_y_of(res)
    _, d = _d.log_ceil(y, n, res.gamma, want_dceil=True)
    return d.cpu().numpy()


def r_distance_device(res) -> torch.Tensor:
    """As r_distance, result left on the device."""
    y, n = _device_y_of(res)
    return _d.log_ceil(y, n, res.gamma, want_r=True)[0]


def critical_gain(g) -> float:
    """1 / spectral radius of the adjacency pattern; +inf when acyclic (resolvent.py:156-165)."""
    w = _d.graph_weights(g)
    n = g.n_vertices
    rho, _, _ = _d.power_iteration(w, indicator=True, tol=1e-6, max_iter=10 * n + 100)
    if rho == 0.0:
        return math.inf
    return 1.0 / rho


def precision_floor(d_max: int) -> float:
    """Smallest gamma whose d_max-th power is still representable (resolvent.py:168-172)."""
    if d_max < 1:
        raise ValueError(f"d_max must be >= 1, got {d_max}")
    return DELTA_MIN ** (1.0 / d_max)


def gamma_bounds(g, d_max: int) -> GammaBounds:
    """Critical gain and precision floor for a known max distance (resolvent.py:175-179)."""
    gc = critical_gain(g)
    floor = precision_floor(d_max)
    return GammaBounds(gc, floor, d_max, floor < gc)


def suggest_gamma(bounds: GammaBounds, safety: float = 0.01) -> float:
    """safety * critical gain, clamped into the valid window (resolvent.py:182-201)."""
    if not bounds.feasible:
        raise InfeasibleGammaError(
            f"no valid gamma: precision floor {bounds.precision_floor_for_dmax:.6g} "
            f">= critical gain {bounds.critical_gain:.6g} at d_max={bounds.d_max_used}"
        )
    if not 0 < safety < 1:
        raise ValueError(f"safety must be in (0, 1), got {safety}")
    gc = min(bounds.critical_gain, 1.0)
    gamma = min(safety * gc, 0.99 * gc)
    return max(gamma, 10.0 * bounds.precision_floor_for_dmax)


def communicability(res) -> float:
    """Sum of all resolvent entries (resolvent.py:204-211; outside the hot path)."""
    if res.health.negative_entries:
        raise ValueError(
            "resolvent has negative entries; communicability is undefined "
            f"at gamma={res.gamma:.6g}"
        )
    return float(res.y.sum())


def is_unweighted(g) -> bool:
    return kind_value(g) == "unweighted"
