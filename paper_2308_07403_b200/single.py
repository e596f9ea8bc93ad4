"""One large unweighted graph from bit-packed adjacency (configs 3 and 5).

The drop-in ``resolvent(g, gamma)`` takes the reference's dense float64 weight
matrix; at N = 32768 that is an 8.6 GB host array. These helpers run the same
pipeline (reference resolvent.py:101-153 with ``with_residual=False``) from the
device bit-packed adjacency (``rdb_build_m_bits`` row format, 128 MB at N =
32768) instead:

  M = I - gamma * A      (K1, rdb_build_m_bits)
  Y = M^-1 in place      (K2, rdb_invert: no-pivot Gauss-Jordan on DMMA; the
                          wide 256-step path for n >= 8192)
  D = ceil(log Y / log gamma) for all pairs (int32) or for sampled source
  columns (K3, rdb_log_ceil / rdb_log_ceil_block).

The pivot record certifies the inverse exactly as the drop-in does
(resolvent._invert_m); an uncertified matrix raises (there is no 8.6 GB
rebuild for the pivoted kernel here).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .linalg import PIVOT_RTOL, SingularMatrixError
from .resolvent import ResolventSingularError


def build_m_bits(bits: torch.Tensor, n: int, gamma: float, out: torch.Tensor | None = None) -> torch.Tensor:
    """n_pad x n_pad M = I - gamma*A (identity padding) from device bits (n, ceil(n/32)) int32."""
    if not 0 < gamma < 1:
        raise ValueError(f"gamma must be in (0, 1), got {gamma}")
    n_pad = L.pad_to_nb(n)
    m = out if out is not None else torch.empty((n_pad, n_pad), dtype=torch.float64, device=bits.device)
    L.check(L.lib().rdb_build_m_bits(bits.data_ptr(), n, n_pad, 1, None, float(gamma), m.data_ptr(), n_pad,
                                     n_pad * n_pad, L.stream_handle()), "rdb_build_m_bits")
    return m


def invert_in_place(m: torch.Tensor, gamma: float) -> L.PivotInfo:
    """Y = M^-1 in place (n_pad x n_pad, contiguous); raises ResolventSingularError
    unless the no-pivot pivots certify a nonsingular M-matrix above PIVOT_RTOL
    (linalg.py:33-38, scale = max|M| = 1)."""
    n_pad = m.shape[0]
    work = torch.empty(L.lib().rdb_invert_workspace_bytes(n_pad, 1), dtype=torch.uint8, device=m.device)
    info = L.pivot_info_tensor(1, m.device)
    L.check(L.lib().rdb_invert(m.data_ptr(), n_pad, m.stride(0), work.data_ptr(), info.data_ptr(),
                               L.stream_handle()), "rdb_invert")
    rec = L.read_pivot_info(info)[0]
    if (rec.flags & (L.RDB_PIV_NONPOS | L.RDB_PIV_NONFINITE)) or not rec.min_pivot >= PIVOT_RTOL:
        raise ResolventSingularError(gamma) from SingularMatrixError(
            f"min pivot {rec.min_pivot:.3e} (flags {rec.flags}); the partial-pivoting path needs the dense W")
    return rec


def d_columns(y: torch.Tensor, n: int, gamma: float, cols) -> torch.Tensor:
    """float64 D[:, cols] (+inf unreachable, 0 on the diagonal): distances from
    the sampled sources, on the device."""
    cols_d = torch.as_tensor(np.asarray(cols, dtype=np.int64), device=y.device)
    ysub = y[:n].index_select(1, cols_d).contiguous()
    k = cols_d.numel()
    d = torch.empty((n, k), dtype=torch.float64, device=y.device)
    L.check(L.lib().rdb_log_ceil_block(ysub.data_ptr(), n, k, k, 0, 0, cols_d.data_ptr(), float(gamma), None,
                                       d.data_ptr(), None, k, None, L.stream_handle()), "rdb_log_ceil_block")
    return d


def d_int32(y: torch.Tensor, n: int, gamma: float, out: torch.Tensor | None = None) -> torch.Tensor:
    """int32 D for all pairs (INT32_MAX unreachable) on the device."""
    d = out if out is not None else torch.empty((n, n), dtype=torch.int32, device=y.device)
    L.check(L.lib().rdb_log_ceil(y.data_ptr(), n, y.stride(0), 0, 1, None, float(gamma), None, None, d.data_ptr(),
                                 n, 0, None, 0, None, L.stream_handle()), "rdb_log_ceil")
    return d
