"""Dense numeric kernels of the path: inversion and power iteration.

Drop-in for pkg/src/rdist/linalg.py (lu_invert :18-39, power_iteration
:57-94, spectral_radius :97-99). Inputs may be numpy arrays (returned
results are numpy arrays, as in the reference) or CUDA tensors (results stay
on the device). All arithmetic runs in the sm_100a kernels of
``librdist_b200.so``; there is no CPU fallback. ``mat_mul`` (linalg.py:42-48,
off the timed path) runs on the same DMMA engine (rdb_gemm_local).
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np
import torch

from . import _device as _d

PIVOT_RTOL = 1e-13  # linalg.py:11


class SingularMatrixError(RuntimeError):
    """Matrix is singular to working precision (a pivot collapsed)."""


class PowerIterationResult(NamedTuple):
    value: float
    converged: bool
    iterations: int


def _check_square(shape) -> None:
    if len(shape) != 2 or shape[0] != shape[1]:
        raise ValueError(f"expected a square matrix, got shape {tuple(shape)}")


def lu_invert(m):
    """Inverse of a square matrix (linalg.py:18-39).

    Raises ValueError for non-square or non-finite input and
    SingularMatrixError when the smallest pivot magnitude is below
    PIVOT_RTOL times the largest input magnitude. Nonsingular M-matrices (the
    resolvent's 1 - gamma^W) are inverted by the no-pivot blocked Gauss-Jordan
    DMMA kernel, whose pivots are LAPACK's diag(U) there; anything else by the
    partial-pivoting Gauss-Jordan kernel.
    """
    if not isinstance(m, torch.Tensor):
        m = np.asarray(m, dtype=np.float64)
    _check_square(m.shape)
    a, on_device = _d.as_device_matrix(m)
    scale, nonfinite, nonz, _ = _d.matrix_stats(a)
    if nonfinite:
        raise ValueError("matrix entries must be finite")
    try:
        y = _d.invert(a, scale, nonz == 0, PIVOT_RTOL)
    except _d.InversionFailure as exc:
        raise SingularMatrixError(str(exc)) from None
    if on_device:
        return y.contiguous()
    return y.cpu().numpy().copy(order="C")


def mat_mul(a, b):
    """Matrix product with an explicit shape check (linalg.py:42-48): C = A B
    on the FP64 DMMA engine (rdb_gemm_local), operands zero-padded to the
    engine's 128 x 128 x 16 tiles. numpy in -> numpy out, CUDA in -> CUDA out."""
    from . import _lib as L

    dev_in = isinstance(a, torch.Tensor) and a.is_cuda
    if not isinstance(a, torch.Tensor):
        a = np.asarray(a, dtype=np.float64)
    if not isinstance(b, torch.Tensor):
        b = np.asarray(b, dtype=np.float64)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ValueError(f"shape mismatch: {tuple(a.shape)} x {tuple(b.shape)}")
    m, k = a.shape
    n = b.shape[1]
    dev = L.device()
    if m == 0 or n == 0 or k == 0:
        out = torch.zeros((m, n), dtype=torch.float64, device=dev)
        return out if dev_in else out.cpu().numpy()
    mp, np_ = L.pad_to_nb(m), L.pad_to_nb(n)
    kp = (k + 15) // 16 * 16
    ap = torch.zeros((mp, kp), dtype=torch.float64, device=dev)
    bp = torch.zeros((kp, np_), dtype=torch.float64, device=dev)
    ap[:m, :k] = torch.as_tensor(a, dtype=torch.float64, device=dev)
    bp[:k, :n] = torch.as_tensor(b, dtype=torch.float64, device=dev)
    cp = torch.empty((mp, np_), dtype=torch.float64, device=dev)
    L.check(L.lib().rdb_gemm_local(ap.data_ptr(), kp, bp.data_ptr(), np_, cp.data_ptr(), np_, mp, np_, kp, -1, -1,
                                   -1, 0, 0, 0, L.stream_handle()), "rdb_gemm_local(mat_mul)")
    out = cp[:m, :n]
    return out.contiguous() if dev_in else out.cpu().numpy().copy(order="C")


def power_iteration(m, tol: float = 1e-6, max_iter: int | None = None) -> PowerIterationResult:
    """Dominant-eigenvalue estimate of a non-negative matrix (linalg.py:57-94).

    Same start vector, geometric-mean estimate, stopping rule and flags as
    the reference; the iteration runs in one cooperative kernel on the GPU.
    """
    if not isinstance(m, torch.Tensor):
        m = np.asarray(m, dtype=np.float64)
    _check_square(m.shape)
    a, _ = _d.as_device_matrix(m)
    _, _, _, negatives = _d.matrix_stats(a)
    if negatives:
        raise ValueError("power iteration expects non-negative entries")
    if tol <= 0:
        raise ValueError(f"tol must be > 0, got {tol}")
    n = a.shape[0]
    if max_iter is None:
        max_iter = 10 * n + 100
    v, c, it = _d.power_iteration(a, indicator=False, tol=tol, max_iter=max_iter)
    return PowerIterationResult(v, c, it)


def spectral_radius(m, tol: float = 1e-6, max_iter: int | None = None) -> float:
    """Largest-magnitude eigenvalue of a non-negative matrix (linalg.py:97-99)."""
    return power_iteration(m, tol=tol, max_iter=max_iter).value
