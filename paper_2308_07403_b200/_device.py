"""Device-side handles and the kernel sequences behind the public API.

Everything here runs on the CUDA device through the C ABI (``_lib``); numpy
arrays are only the host-side inputs/outputs the reference API trades in.
"""

from __future__ import annotations

import math
import weakref

import numpy as np
import torch

from . import _lib as L

# Graph weights are immutable (the reference sets them read-only), so their
# device copy can be cached for the lifetime of the Graph object.
_weights_cache: dict[int, torch.Tensor] = {}


def _evict(key: int) -> None:
    _weights_cache.pop(key, None)


def graph_weights(g) -> torch.Tensor:
    """Device float64 copy of ``g.weights`` (cached per live Graph object)."""
    key = id(g)
    t = _weights_cache.get(key)
    if t is not None:
        return t
    dev = L.device()
    w = np.array(g.weights, dtype=np.float64, order="C", copy=True)
    t = torch.from_numpy(w).to(dev, non_blocking=False)
    try:
        weakref.finalize(g, _evict, key)
        _weights_cache[key] = t
    except TypeError:  # not weak-referenceable: do not cache
        pass
    return t


def as_device_matrix(m) -> tuple[torch.Tensor, bool]:
    """(contiguous float64 CUDA tensor, came_from_torch)."""
    dev = L.device()
    if isinstance(m, torch.Tensor):
        return m.to(device=dev, dtype=torch.float64).contiguous(), True
    a = np.ascontiguousarray(np.asarray(m, dtype=np.float64))
    return torch.from_numpy(a).to(dev), False


def matrix_stats(a: torch.Tensor) -> tuple[float, int, int, int]:
    """(max|a|, non-finite count, Z-pattern violations, negatives)."""
    n = a.shape[0]
    stats = torch.zeros(4, dtype=torch.float64, device=a.device)
    L.check(L.lib().rdb_matrix_stats(a.data_ptr(), n, a.stride(0), stats.data_ptr(), L.stream_handle()),
            "rdb_matrix_stats")
    s = stats.cpu().tolist()
    return s[0], int(s[1]), int(s[2]), int(s[3])


def build_m(w: torch.Tensor, n: int, gamma: float, n_pad: int | None = None, mode: int = L.RDB_BUILD_M) -> torch.Tensor:
    """K1: M = I - gamma^W (padded to n_pad with identity) or X = gamma^W."""
    if mode == L.RDB_BUILD_M:
        n_pad = L.pad_to_nb(n) if n_pad is None else n_pad
        out = torch.empty((n_pad, n_pad), dtype=torch.float64, device=w.device)
    else:
        n_pad = n
        out = torch.empty((n, n), dtype=torch.float64, device=w.device)
    L.check(
        L.lib().rdb_build_m(w.data_ptr(), w.stride(0), 0, n, n_pad, 1, None, float(gamma), mode,
                            out.data_ptr(), out.stride(0), 0, L.stream_handle()),
        "rdb_build_m",
    )
    return out


class InversionFailure(Exception):
    """Internal: carries the reference-style singularity message."""

    def __init__(self, min_pivot: float, scale: float):
        super().__init__(f"singular to working precision (min pivot {min_pivot:.3e}, scale {scale:.3e})")
        self.min_pivot = min_pivot
        self.scale = scale


def invert_padded_nopivot(a_pad: torch.Tensor) -> L.PivotInfo:
    """K2 in place on an n_pad x n_pad (identity-padded) matrix; returns the pivot record."""
    n_pad = a_pad.shape[0]
    work = torch.empty(L.lib().rdb_invert_workspace_bytes(n_pad, 1), dtype=torch.uint8, device=a_pad.device)
    info = L.pivot_info_tensor(1, a_pad.device)
    L.check(L.lib().rdb_invert(a_pad.data_ptr(), n_pad, a_pad.stride(0), work.data_ptr(), info.data_ptr(),
                               L.stream_handle()), "rdb_invert")
    return L.read_pivot_info(info)[0]


def invert_pivoted(a: torch.Tensor) -> L.PivotInfo:
    n = a.shape[0]
    work = torch.empty(L.lib().rdb_invert_pivoted_workspace_bytes(n), dtype=torch.uint8, device=a.device)
    info = L.pivot_info_tensor(1, a.device)
    L.check(L.lib().rdb_invert_pivoted(a.data_ptr(), n, a.stride(0), work.data_ptr(), info.data_ptr(),
                                       L.stream_handle()), "rdb_invert_pivoted")
    return L.read_pivot_info(info)[0]


def pad_copy(a: torch.Tensor, n_pad: int) -> torch.Tensor:
    n = a.shape[0]
    if n == n_pad:
        return a.clone()
    out = torch.empty((n_pad, n_pad), dtype=torch.float64, device=a.device)
    out[:n, :n].copy_(a)
    L.check(L.lib().rdb_pad_identity(out.data_ptr(), n, n_pad, out.stride(0), 0, 1, L.stream_handle()),
            "rdb_pad_identity")
    return out


def invert(a: torch.Tensor, scale: float, z_matrix: bool, pivot_rtol: float) -> torch.Tensor:
    """Y = a^-1 for a square finite device matrix (a is not modified).

    Z-matrices go through the no-pivot DMMA kernel; its pivots certify the
    result (all positive => nonsingular M-matrix, where partial pivoting is
    unnecessary). Without that certificate, or when a no-pivot pivot falls
    below the tolerance, the partial-pivoting kernel runs and its pivots decide.
    Raises InversionFailure on the reference's rule min|pivot| < rtol*scale
    (linalg.py:33-38).
    """
    n = a.shape[0]
    tol = pivot_rtol * scale
    if scale == 0.0:
        raise InversionFailure(0.0, scale)
    if z_matrix:
        n_pad = L.pad_to_nb(n)
        y = pad_copy(a, n_pad)
        rec = invert_padded_nopivot(y)
        if not (rec.flags & (L.RDB_PIV_NONPOS | L.RDB_PIV_NONFINITE)) and rec.min_pivot >= tol:
            return y[:n, :n] if n_pad != n else y
    y = a.clone()
    rec = invert_pivoted(y)
    if (rec.flags & L.RDB_PIV_NONFINITE) or not (rec.min_pivot >= tol):
        raise InversionFailure(rec.min_pivot, scale)
    return y


def log_ceil(y: torch.Tensor, n: int, gamma: float, *, want_r: bool = False, want_dceil: bool = False,
             reachable: torch.Tensor | None = None, counters: torch.Tensor | None = None):
    """K3 over the leading n x n block of y; returns (R or None, Dceil or None)."""
    dev = y.device
    r = torch.empty((n, n), dtype=torch.float64, device=dev) if want_r else None
    d = torch.empty((n, n), dtype=torch.float64, device=dev) if want_dceil else None
    ldo = n
    L.check(
        L.lib().rdb_log_ceil(y.data_ptr(), n, y.stride(0), 0, 1, None, float(gamma), L.ptr(r), L.ptr(d), None,
                             ldo, 0, L.ptr(reachable), n if reachable is not None else 0, L.ptr(counters),
                             L.stream_handle()),
        "rdb_log_ceil",
    )
    return r, d


def residual(m_pad: torch.Tensor, y_pad: torch.Tensor) -> float:
    out = torch.zeros(1, dtype=torch.float64, device=m_pad.device)
    L.check(L.lib().rdb_residual(m_pad.data_ptr(), m_pad.stride(0), y_pad.data_ptr(), y_pad.stride(0),
                                 m_pad.shape[0], out.data_ptr(), L.stream_handle()), "rdb_residual")
    return float(out.item())


def power_iteration(m: torch.Tensor, indicator: bool, tol: float, max_iter: int) -> tuple[float, bool, int]:
    n = m.shape[0]
    work = torch.empty(L.lib().rdb_power_workspace_bytes(n), dtype=torch.uint8, device=m.device)
    res = torch.zeros(3, dtype=torch.float64, device=m.device)
    L.check(L.lib().rdb_power_iteration(m.data_ptr(), n, m.stride(0), 1 if indicator else 0, float(tol),
                                        int(max_iter), work.data_ptr(), res.data_ptr(), L.stream_handle()),
            "rdb_power_iteration")
    v, c, it = res.cpu().tolist()
    return v, bool(c != 0.0), int(it)


def count_edges(w: torch.Tensor) -> int:
    out = torch.zeros(1, dtype=torch.int64, device=w.device)
    L.check(L.lib().rdb_count_edges(w.data_ptr(), w.shape[0], w.stride(0), out.data_ptr(), L.stream_handle()),
            "rdb_count_edges")
    return int(out.item())


def next_hop(w: torch.Tensor, dist_rows: torch.Tensor, targets: torch.Tensor, nnz: int | None = None) -> torch.Tensor:
    """K6: next[r][j] for target targets[r] using dist_rows[r] (device tensors)."""
    n = w.shape[0]
    if nnz is None:
        nnz = count_edges(w)
    nt = targets.shape[0]
    out = torch.empty((nt, n), dtype=torch.int32, device=w.device)
    work = torch.empty(max(1, L.lib().rdb_next_hop_workspace_bytes(n, nnz, nt)), dtype=torch.uint8, device=w.device)
    L.check(
        L.lib().rdb_next_hop(w.data_ptr(), w.stride(0), dist_rows.data_ptr(), dist_rows.stride(0), n, nnz,
                             targets.data_ptr(), nt, out.data_ptr(), out.stride(0), work.data_ptr(),
                             L.stream_handle()),
        "rdb_next_hop",
    )
    return out


def finite_or_nan(x: float) -> float:
    return x if math.isfinite(x) else math.nan
