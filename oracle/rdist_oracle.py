"""CPU oracle for the R-distance hot path — TEST INFRASTRUCTURE ONLY.

A restatement, in numpy/scipy, of the reference algorithm for the path
(arXiv 2308.07403's ``rdist`` package, /root/reference/pkg/src/rdist/). It is
the checker the CUDA path is compared against and the CPU baseline bench.py
times. Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import it; the product
package never does (it has no CPU fallback).

Pinning: every function here was checked against outputs of the reference
itself, run in the build container (tests/golden/make_golden.py writes them
to tests/golden/*.npz; tests/test_oracle_golden.py compares). The arithmetic
of the reference lives in numpy and scipy (LAPACK getrf/getrs via
scipy.linalg.lu_factor / lu_solve, OpenBLAS); those are called here exactly
as the reference calls them, so the oracle reproduces its results bit for
bit on the same machine and thread count.
"""

from __future__ import annotations

import math
import os
import statistics
import time
import warnings

import numpy as np
import scipy.linalg

PIVOT_RTOL = 1e-13  # linalg.py:11
NEGATIVE_ENTRY_TOL = -1e-12  # resolvent.py:26


class OracleSingular(RuntimeError):
    pass


def build_x(w: np.ndarray, gamma: float) -> np.ndarray:
    """gamma**W entry-wise, gamma**inf = 0 (resolvent.py:90-98)."""
    if not 0 < gamma < 1:
        raise ValueError(f"gamma must be in (0, 1), got {gamma}")
    return np.power(gamma, w)


def lu_invert(m: np.ndarray) -> np.ndarray:
    """LAPACK getrf with partial pivoting, singularity rule, getrs(I) (linalg.py:18-39)."""
    m = np.asarray(m, dtype=np.float64)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {m.shape}")
    if not np.isfinite(m).all():
        raise ValueError("matrix entries must be finite")
    scale = float(np.abs(m).max())
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        lu, piv = scipy.linalg.lu_factor(m, check_finite=False)
    pivots = np.abs(np.diagonal(lu))
    if scale == 0.0 or (pivots < PIVOT_RTOL * scale).any():
        raise OracleSingular(f"min pivot {pivots.min():.3e}, scale {scale:.3e}")
    return scipy.linalg.lu_solve((lu, piv), np.eye(m.shape[0]), check_finite=False)


def resolvent_y(w: np.ndarray, gamma: float) -> np.ndarray:
    """Y = (I - gamma**W)^-1 (resolvent.py:114-119)."""
    n = w.shape[0]
    return lu_invert(np.eye(n) - build_x(w, gamma))


def health(y: np.ndarray, reachable: np.ndarray | None = None):
    """(negative_entries, underflow_zeros) as resolvent.py:120-124 computes them."""
    negative = bool((y < NEGATIVE_ENTRY_TOL).any())
    under = None
    if reachable is not None:
        off = ~np.eye(y.shape[0], dtype=bool)
        under = int(((y == 0.0) & reachable & off).sum())
    return negative, under


def residual(m: np.ndarray, y: np.ndarray) -> float:
    """max |M Y - I| (resolvent.py:125-127)."""
    return float(np.abs(m @ y - np.eye(m.shape[0])).max())


def r_distance(y: np.ndarray, gamma: float) -> np.ndarray:
    """log Y / log gamma where Y > 0, else +inf; zero diagonal (resolvent.py:131-143)."""
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(y > 0, np.log(y) / math.log(gamma), np.inf)
    np.fill_diagonal(r, 0.0)
    return r


def rounded_r_distance(y: np.ndarray, gamma: float) -> np.ndarray:
    """ceil(R), no nudge (resolvent.py:146-153)."""
    return np.ceil(r_distance(y, gamma))


def run_rdist(w: np.ndarray, gamma: float, unweighted: bool = True) -> np.ndarray:
    """The reference's timed closure (experiments.py:305-310): resolvent(with_residual=False)
    computes its health flags too (resolvent.py:120-124), then r_distance and ceil."""
    y = resolvent_y(w, gamma)
    health(y)
    r = r_distance(y, gamma)
    return np.ceil(r) if unweighted else r


def d_to_int32(d: np.ndarray) -> np.ndarray:
    """fp64 D with +inf -> int32 with INT32_MAX (the device output format)."""
    out = np.full(d.shape, 2147483647, dtype=np.int32)
    fin = np.isfinite(d)
    out[fin] = d[fin].astype(np.int32)
    return out


def power_iteration(m: np.ndarray, tol: float = 1e-6, max_iter: int | None = None):
    """(value, converged, iterations) exactly as linalg.py:57-94."""
    m = np.asarray(m, dtype=np.float64)
    n = m.shape[0]
    if max_iter is None:
        max_iter = 10 * n + 100
    v = np.ones(n) / np.sqrt(n)
    prev_ratio = prev_est = None
    est = 0.0
    for it in range(1, max_iter + 1):
        w = m @ v
        ratio = float(np.linalg.norm(w))
        if ratio == 0.0:
            return 0.0, True, it
        est = ratio if prev_ratio is None else float(np.sqrt(ratio * prev_ratio))
        if prev_est is not None and abs(est - prev_est) < tol:
            return est, True, it
        prev_ratio, prev_est = ratio, est
        v = w / ratio
    return est, False, max_iter


def next_hop_table(w: np.ndarray, dist: np.ndarray, targets=None) -> np.ndarray:
    """The greedy step of navigation.py:62-69 for every (target, vertex):
    next[t][j] = first argmin over ascending successors k of j of
    W[k][j] + dist[t][k]; -1 if j == t, no successor, or non-finite best."""
    n = w.shape[0]
    targets = np.arange(n) if targets is None else np.asarray(targets)
    out = np.full((len(targets), n), -1, dtype=np.int32)
    for j in range(n):
        succ = np.flatnonzero(np.isfinite(w[:, j]))
        if succ.size == 0:
            continue
        scores = w[succ, j][None, :] + dist[np.ix_(targets, succ)]
        best = np.argmin(scores, axis=1)
        ok = np.isfinite(scores[np.arange(len(targets)), best]) & (targets != j)
        out[ok, j] = succ[best[ok]]
    return out


def greedy_descent(w: np.ndarray, dist: np.ndarray, start: int, goal: int, max_steps: int | None = None):
    """(vertices, length, reached, steps) as navigation.py:35-74."""
    n = w.shape[0]
    if max_steps is None:
        max_steps = 4 * n
    path, length, cur, steps = [start], 0.0, start, 0
    while cur != goal and steps < max_steps:
        succ = np.flatnonzero(np.isfinite(w[:, cur]))
        if succ.size == 0:
            break
        scores = w[succ, cur] + dist[goal, succ]
        best = int(np.argmin(scores))
        if not np.isfinite(scores[best]):
            break
        length += float(w[succ[best], cur])
        cur = int(succ[best])
        path.append(cur)
        steps += 1
    return path, length, cur == goal, steps


def bfs_apsp(w: np.ndarray) -> np.ndarray:
    """Exact unweighted distances, level-synchronous (oracles.py:22-41)."""
    n = w.shape[0]
    a = np.isfinite(w).astype(np.float64)
    dist = np.full((n, n), np.inf)
    np.fill_diagonal(dist, 0.0)
    frontier = np.eye(n)
    for level in range(1, n):
        frontier = (a @ frontier > 0).astype(np.float64)
        newly = (frontier > 0) & np.isinf(dist)
        if not newly.any():
            break
        dist[newly] = level
    return dist


def floyd_warshall(w: np.ndarray) -> np.ndarray:
    """The classic vectorised k-loop (oracles.py:44-50)."""
    d = np.array(w, dtype=np.float64, copy=True)
    np.fill_diagonal(d, 0.0)
    for k in range(d.shape[0]):
        np.minimum(d, np.add.outer(d[:, k], d[k, :]), out=d)
    return d


def global_accuracy(est: np.ndarray, exact: np.ndarray) -> float:
    """Share of finite off-diagonal exact pairs the estimate hits exactly (navigation.py:77-88)."""
    keep = np.isfinite(exact)
    np.fill_diagonal(keep, False)
    total = int(keep.sum())
    return float("nan") if total == 0 else float(np.count_nonzero(est[keep] == exact[keep]) / total)


def local_accuracy(w: np.ndarray, est: np.ndarray, exact: np.ndarray, atol: float = 0.0) -> float:
    """Share of (goal, node) pairs whose first-minimum successor by the estimate
    is also a closest successor by the exact distances (navigation.py:91-134)."""
    n = w.shape[0]
    succ = np.isfinite(w)  # succ[k, i]: edge i -> k
    has_succ = succ.any(axis=0)
    total = hits = 0
    for t in range(n):
        nodes = np.flatnonzero(np.isfinite(exact[t]) & has_succ & (np.arange(n) != t))
        if nodes.size == 0:
            continue
        e = np.where(succ[:, nodes], est[t][:, None], np.inf)
        x = np.where(succ[:, nodes], exact[t][:, None], np.inf)
        pick = e.argmin(axis=0)  # lowest index on ties, first NaN wins (numpy argmin)
        chosen = e[pick, np.arange(nodes.size)]
        hits += int(np.count_nonzero(np.isfinite(chosen) & (exact[t, pick] <= x.min(axis=0) + atol)))
        total += nodes.size
    return float("nan") if total == 0 else hits / total


def sampled_columns_d(m_fortran: np.ndarray, cols: np.ndarray, gamma: float) -> np.ndarray:
    """Config-5 restatement: lu_factor(M) as linalg.py:32,
    then lu_solve on identity columns E_S; returns ceil(R) for those columns
    (D[:, S], i.e. distances from the sampled sources). Overwrites m."""
    n = m_fortran.shape[0]
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        lu, piv = scipy.linalg.lu_factor(m_fortran, overwrite_a=True, check_finite=False)
    e = np.zeros((n, len(cols)))
    e[cols, np.arange(len(cols))] = 1.0
    ycols = scipy.linalg.lu_solve((lu, piv), e, check_finite=False)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(ycols > 0, np.log(ycols) / math.log(gamma), np.inf)
    r[cols, np.arange(len(cols))] = 0.0
    return np.ceil(r)


def median_time(fn, runs: int) -> float:
    """The reference timing protocol (experiments.py:263-270)."""
    fn()
    times = []
    for _ in range(runs):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    return statistics.median(times)


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        info = threadpool_info()
        return max((i.get("num_threads", 1) for i in info), default=os.cpu_count() or 1)
    except Exception:  # noqa: BLE001 - informational only
        return os.cpu_count() or 1
