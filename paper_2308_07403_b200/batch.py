"""Batched all-pairs distances for many independent unweighted graphs.

The config-2 workload: the reference's timed closure ``run_rdist``
(pkg/src/rdist/experiments.py:305-310: resolvent(g, gamma,
with_residual=False) -> r_distance -> ceil) applied to a batch of graphs
with per-graph gains, as one device pipeline per chunk: bit-packed adjacency
-> M = I - gamma*A (K1) -> batched Gauss-Jordan inverse (K2) -> int32
D = ceil(log Y / log gamma) (K3), via ``rdb_apsp_bits_batched``.

int32 D uses INT32_MAX for unreachable pairs (the reference's +inf) and 0 on
the diagonal. ``d_dtype="uint8"`` selects the compact form (rdb_log_ceil_d8):
the same D wherever 0 <= D <= 254, 255 for unreachable pairs, a quarter of the
int32 bytes over PCIe; a graph with a D outside that range is counted on the
device and redone in int32 (:meth:`APSPBatchEngine.wait` widens the batch), so
the result is never lossy. A graph whose no-pivot inverse is not certified
(gamma past the critical gain, or a pivot below tolerance) is recomputed
through the partial-pivoting path, which raises ResolventSingularError
(naming the graph) exactly where the reference's LAPACK path would.

:class:`APSPBatchEngine` owns reusable device and pinned host buffers (the
serving form: host bits in, host int32 D out, copies overlapped with the
kernels on two streams); :func:`rounded_r_distance_batch` is the one-shot
convenience wrapper.
"""

from __future__ import annotations

from dataclasses import dataclass

import os

import numpy as np
import torch

from . import _lib as L
from .linalg import PIVOT_RTOL, SingularMatrixError
from .resolvent import ResolventSingularError

UNREACHABLE = L.INT32_SENTINEL
UNREACHABLE_D8 = L.RDB_D8_UNREACHABLE
D_DTYPES = {"int32": torch.int32, "uint8": torch.uint8}


def bits_from_edge_list(edges, device=None) -> torch.Tensor:
    """Device bit-packed adjacency (n, ceil(n/32)) int32 of an unweighted
    EdgeList (graphs.py wire format), built on the GPU (rdb_edges_to_bits).
    Same validation as graph_from_edge_list: range, self-loops, duplicates."""
    n = int(edges.vertex_count)
    if n < 1:
        raise ValueError("vertex_count must be >= 1")
    e = np.asarray([(s, d) for s, d, _ in edges.edges], dtype=np.int64).reshape(-1, 2)
    w = np.asarray([w for _, _, w in edges.edges], dtype=np.float64)
    if e.size:
        if e.min() < 0 or e.max() >= n:
            raise ValueError(f"edge out of range for {n} vertices")
        if (e[:, 0] == e[:, 1]).any():
            raise ValueError("self-loop in edge list")
        if np.unique(e[:, 0] * n + e[:, 1]).size != e.shape[0]:
            raise ValueError("duplicate edge in edge list")
        if not np.all(w == 1.0):
            raise ValueError("bits_from_edge_list needs an unweighted edge list (all weights 1)")
    dev = device or L.device()
    bits = torch.empty((n, (n + 31) // 32), dtype=torch.int32, device=dev)
    src = torch.from_numpy(np.ascontiguousarray(e[:, 0], dtype=np.int32)).to(dev)
    dst = torch.from_numpy(np.ascontiguousarray(e[:, 1], dtype=np.int32)).to(dev)
    L.check(L.lib().rdb_edges_to_bits(src.data_ptr() if e.size else None, dst.data_ptr() if e.size else None,
                                      int(e.shape[0]), n, bits.data_ptr(), L.stream_handle()), "rdb_edges_to_bits")
    return bits


def decode_d8(d8: np.ndarray) -> np.ndarray:
    """uint8 D -> int32 D (255 -> INT32_MAX)."""
    d = d8.astype(np.int32)
    d[d8 == L.RDB_D8_UNREACHABLE] = UNREACHABLE
    return d


@dataclass
class BatchBuffers:
    """Device buffers for up to ``chunk`` graphs of ``n`` vertices."""

    n: int
    chunk: int
    bits: torch.Tensor
    gammas: torch.Tensor
    m: torch.Tensor
    work: torch.Tensor
    info: torch.Tensor
    d: torch.Tensor
    counters: torch.Tensor

    @classmethod
    def allocate(cls, n: int, chunk: int, dev: torch.device, d_dtype: str = "int32") -> "BatchBuffers":
        n_pad = L.pad_to_nb(n)
        wpr = (n + 31) // 32
        return cls(
            n=n,
            chunk=chunk,
            bits=torch.empty((chunk, n, wpr), dtype=torch.int32, device=dev),
            gammas=torch.empty(chunk, dtype=torch.float64, device=dev),
            m=torch.empty((chunk, n_pad, n_pad), dtype=torch.float64, device=dev),
            work=torch.empty(L.lib().rdb_invert_workspace_bytes(n_pad, chunk), dtype=torch.uint8, device=dev),
            info=L.pivot_info_tensor(chunk, dev),
            d=torch.empty((chunk, n, n), dtype=D_DTYPES[d_dtype], device=dev),
            counters=torch.zeros((chunk, L.RDB_NCOUNTERS), dtype=torch.int64, device=dev),
        )

    @property
    def compact(self) -> bool:
        return self.d.dtype == torch.uint8

    @property
    def n_pad(self) -> int:
        return self.m.shape[-1]

    # the three stages separately (bench.py times each kernel family)
    def stage_build(self, count: int, stream: int) -> None:
        L.check(L.lib().rdb_build_m_bits(self.bits.data_ptr(), self.n, self.n_pad, count, self.gammas.data_ptr(),
                                         0.0, self.m.data_ptr(), self.n_pad, self.n_pad * self.n_pad, stream),
                "rdb_build_m_bits")

    def stage_invert(self, count: int, stream: int) -> None:
        """K2 with the block pattern from the adjacency bits (as the apsp pipeline)."""
        L.check(L.lib().rdb_invert_batched_bits(self.m.data_ptr(), self.n_pad, self.n_pad, self.n_pad * self.n_pad,
                                                count, self.bits.data_ptr(), self.n, self.work.data_ptr(),
                                                self.info.data_ptr(), stream),
                "rdb_invert_batched_bits")

    def stage_invert_generic(self, count: int, stream: int) -> None:
        """K2 through the generic entry point (block pattern by scanning M)."""
        L.check(L.lib().rdb_invert_batched(self.m.data_ptr(), self.n_pad, self.n_pad, self.n_pad * self.n_pad,
                                           count, self.work.data_ptr(), self.info.data_ptr(), stream),
                "rdb_invert_batched")

    def stage_log_ceil(self, count: int, stream: int) -> None:
        log_ceil_call(self.m, self.n, count, self.gammas, self.d, self.counters, stream)


def apsp_call(bits: torch.Tensor, n: int, count: int, gammas: torch.Tensor, m: torch.Tensor, work: torch.Tensor,
              info: torch.Tensor, d: torch.Tensor, counters: torch.Tensor, stream: int) -> None:
    """One rdb_apsp_bits_batched[_d8] call (K1 -> K2 -> K3); the D dtype picks the entry point."""
    fn, name = ((L.lib().rdb_apsp_bits_batched_d8, "rdb_apsp_bits_batched_d8") if d.dtype == torch.uint8
                else (L.lib().rdb_apsp_bits_batched, "rdb_apsp_bits_batched"))
    L.check(fn(bits.data_ptr(), n, count, gammas.data_ptr(), m.data_ptr(), work.data_ptr(), info.data_ptr(),
               d.data_ptr(), counters.data_ptr(), stream), name)


def log_ceil_call(m: torch.Tensor, n: int, count: int, gammas: torch.Tensor, d: torch.Tensor,
                  counters: torch.Tensor, stream: int) -> None:
    """K3 over ``count`` padded inverses in ``m`` into D (int32 or uint8 by dtype)."""
    n_pad = m.shape[-1]
    if d.dtype == torch.uint8:
        L.check(L.lib().rdb_log_ceil_d8(m.data_ptr(), n, n_pad, n_pad * n_pad, count, gammas.data_ptr(), 0.0,
                                        d.data_ptr(), n, n * n, counters.data_ptr(), stream), "rdb_log_ceil_d8")
    else:
        L.check(L.lib().rdb_log_ceil(m.data_ptr(), n, n_pad, n_pad * n_pad, count, gammas.data_ptr(), 0.0, None,
                                     None, d.data_ptr(), n, n * n, None, 0, counters.data_ptr(), stream),
                "rdb_log_ceil")


def run_chunk(buf: BatchBuffers, count: int, stream: int | None = None) -> None:
    """Launch K1 -> K2 -> K3 for the first ``count`` graphs held in ``buf``
    (uint8 D: the range counters must be zero; :func:`d8_range_errors` reads them)."""
    apsp_call(buf.bits, buf.n, count, buf.gammas, buf.m, buf.work, buf.info, buf.d, buf.counters,
              L.stream_handle() if stream is None else stream)


class CapturedPipeline:
    """One K1 -> K2 -> K3 call (:func:`run_chunk`, ~300 kernels on the caller's
    stream and the library's internal sub-batch / look-ahead streams, which the
    library joins back with events) captured once into a CUDA graph and
    replayed on the current stream: no per-kernel host launch cost, and the
    device-side gaps between dependent kernels shrink. The buffers are fixed at
    capture; refill ``buf.bits`` / ``buf.gammas`` in place between replays."""

    def __init__(self, buf: "BatchBuffers", count: int):
        self.buf, self.count = buf, count
        run_chunk(buf, count)  # eager first: library setup (streams, attributes) stays outside the capture
        torch.cuda.synchronize()
        self.graph = None
        if os.environ.get("RDB_PIPELINE_EAGER") == "1":  # debugging: every replay is an eager call
            return
        try:  # keep the cudaGraph_t so kernel_nodes() can inspect it
            self.graph = torch.cuda.CUDAGraph(keep_graph=True)
        except TypeError:
            self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            run_chunk(buf, count, torch.cuda.current_stream().cuda_stream)
        if hasattr(self.graph, "instantiate"):
            self.graph.instantiate()

    def replay(self) -> None:
        if self.graph is None:
            run_chunk(self.buf, self.count, torch.cuda.current_stream().cuda_stream)
            return
        self.graph.replay()

    def kernel_nodes(self) -> int:
        """Kernel launches one replay performs, counted from the captured graph's
        nodes (cudaGraphGetNodes / cudaGraphNodeGetType)."""
        from cuda.bindings import runtime as rt

        g = self.graph.raw_cuda_graph()
        err, _, count = rt.cudaGraphGetNodes(g, 0)
        err, nodes, count = rt.cudaGraphGetNodes(g, count)
        kernels = 0
        for nd in nodes[:count]:
            err, t = rt.cudaGraphNodeGetType(nd)
            kernels += t == rt.cudaGraphNodeType.cudaGraphNodeTypeKernel
        return int(kernels)


def d8_range_errors(counters: torch.Tensor) -> np.ndarray:
    """Indices of graphs whose uint8 D had an entry outside [0, 254] (redo them in int32)."""
    c = counters.cpu().numpy().reshape(-1, L.RDB_NCOUNTERS)[:, L.RDB_CNT_D8_RANGE]
    return np.nonzero(c)[0]


PLAN_MAX_NT = 64  # block-sparse plan limit (csrc/gj_invert.cu PLAN_MAX_NT)
SPLIT_MIN_BATCH, SPLIT_PARTS = 64, 2  # csrc/gj_invert.cu defaults (RDB_GJ_SPLIT_MIN / RDB_GJ_SPLIT_PARTS)


def _dw_launches(bands: int, s0: bool, helpers: bool) -> int:
    """Kernels of one one-level dense-wide inversion (dw_part) of a part:
    the first band inverse (6), per band its row panel and update (+ the
    look-ahead's first update, the next band's inverse (6) and a helper launch
    for every band but the last); with a sparse first step its row panel and
    two row ranges of its update (the second only when there are rows past
    the next band)."""
    n = 6 + 2 * bands + 7 * (bands - 1) + (bands - 1 if helpers else 0)
    return n + (2 + (1 if bands > 2 else 0) if s0 else 0)


def launches_per_call(n: int, batch: int) -> int:
    """Kernels one rdb_apsp_bits_batched[_d8] call launches with the default
    knobs (checked against the kernel nodes of a captured call: 159 for the
    config-2 batch): band detection, K1, the strip patterns, the dense-wide
    classification and its edge counts before K1 (one per level), the banded
    factor and chain, K3; per sub-batch the block-sparse plan (3) with 3 per
    panel (P1, P2, U, launched even when their lists are empty), the gathers
    and list splits of the sparse first steps (2 per level) and the dense-wide
    inversion: one-level (:func:`_dw_launches`) or, for n = 1024, two-level
    (two 512 x 512 one-level inversions, the outer steps' row panel and update
    (2 each) and the sparse outer step's row panel and update (2))."""
    nt = L.pad_to_nb(n) // L.RDB_NB
    parts = SPLIT_PARTS if batch >= SPLIT_MIN_BATCH and batch >= 4 * SPLIT_PARTS else 1
    plan = batch > 1 and nt <= PLAN_MAX_NT
    if not plan:
        return 2 + parts * 3 * nt
    dw = nt >= 4 and nt % 2 == 0 and batch >= 2 * parts and not _off("RDB_GJ_DW")
    s0 = dw and not _off("RDB_GJ_DW_S0")
    helpers = not _off("RDB_GJ_DW_HELPER")
    two = dw and two_level(n, batch)
    levels = 2 if two else 1
    if not dw:
        per_part = 0
    elif two:
        per_part = (2 * levels if s0 else 0) + _dw_launches(2, s0, helpers) + _dw_launches(2, False, helpers) + 4 + (
            2 if s0 else 0)
    else:
        per_part = (2 if s0 else 0) + _dw_launches(nt // 2, s0, helpers)
    return (1 + 1 + 1 + (1 if dw else 0) + (levels if s0 else 0) + 2 + 1
            + parts * (3 + 3 * nt + per_part))


STRIPS = 8  # 16-column strips (engine k-chunks) per 128-column block


def _masks(nz: np.ndarray) -> np.ndarray:
    return (nz * (1 << np.arange(STRIPS))).sum(axis=-1).astype(np.uint8)


def strip_pattern(bits: np.ndarray, n: int) -> np.ndarray:
    """Host restatement of strip_pattern_bits_kernel: (batch, 2, nt, nt)
    uint8; [b, 0, I, J] bit s = block (I, J) holds an edge in its 16-column
    strip s, [b, 1, I, J] bit s = in its 16-row strip s (bit-packed rows as
    rdb_build_m_bits takes them)."""
    bits = np.asarray(bits).view(np.uint32)
    batch = bits.shape[0]
    nt = L.pad_to_nb(n) // L.RDB_NB
    nb = L.RDB_NB
    wpr = (n + 31) // 32
    words = bits.reshape(batch, n, wpr)
    halves = np.stack([(words & 0xFFFF) != 0, (words >> 16) != 0], axis=3).reshape(batch, n, 2 * wpr)
    halves = np.concatenate([halves, np.zeros((batch, n, nt * STRIPS - 2 * wpr), bool)], axis=2)
    rows = np.concatenate([halves, np.zeros((batch, nt * nb - n, nt * STRIPS), bool)], axis=1)
    r5 = rows.reshape(batch, nt, STRIPS, nb // STRIPS, nt, STRIPS)  # (b, I, row strip, row, J, col strip)
    col = _masks(r5.any(axis=(2, 3)))                               # (b, I, J)
    row = _masks(r5.any(axis=(3, 5)).transpose(0, 1, 3, 2))        # (b, I, J)
    return np.stack([col, row], axis=1)


def gj_plan_chunks(pattern: np.ndarray) -> np.ndarray:
    """Host restatement of gj_plan_kernel's symbolic Gauss-Jordan
    (csrc/gj_invert.cu): per matrix, the 128 x 128 x 16 k-chunks each kernel
    family executes, columns (P1, P2, U). ``pattern``: (batch, 2, nt, nt)
    column / row strip masks, or (batch, nt, nt) column masks (row masks then
    full on every non-zero block, as strip_pattern_m_kernel). Step p: P2 runs
    every non-zero A_pJ (J != p) over the k-chunks first..last non-zero row
    strip of A_pJ; U runs, for every non-zero A_Ip (I != p), the tiles J of
    P2 plus the panel column over the k-chunks first..last non-zero column
    strip of A_Ip; fill C(A_IJ) |= C(A_pJ), R(A_IJ) |= R(A_Ip); then D A_pJ
    has full rows, A_Ip D full columns, A_pp full. P1 counts as a full tile.
    A dense pattern gives 8 nt^3 chunks = 2 n^3 flop."""
    pattern = np.asarray(pattern, dtype=np.uint8)
    if pattern.ndim == 3:
        pattern = np.stack([pattern, np.where(pattern != 0, 0xFF, 0).astype(np.uint8)], axis=1)
    C = pattern[:, 0].copy()
    R = pattern[:, 1].copy()
    batch, nt, _ = C.shape
    idx = np.arange(nt)
    C[:, idx, idx] = 0xFF
    R[:, idx, idx] = 0xFF
    out = np.zeros((batch, 3), np.int64)
    out[:, 0] = nt * STRIPS
    span = np.zeros(256, np.int64)
    for m in range(1, 256):
        nzb = [s for s in range(STRIPS) if m >> s & 1]
        span[m] = nzb[-1] - nzb[0] + 1
    for k in range(nt):
        rowp = (C[:, k, :] != 0) & (idx != k)
        colp = (C[:, :, k] != 0) & (idx != k)
        nrp = rowp.sum(axis=1)
        out[:, 1] += (span[R[:, k, :]] * rowp).sum(axis=1)
        out[:, 2] += (span[C[:, :, k]] * colp).sum(axis=1) * (nrp + 1)
        R[:, k, :] = np.where(rowp, 0xFF, R[:, k, :])
        both = colp[:, :, None] & rowp[:, None, :]
        C |= np.where(both, C[:, k, None, :], 0).astype(np.uint8)
        R |= np.where(both, R[:, :, k, None], 0).astype(np.uint8)
        C[:, :, k] = np.where(colp, 0xFF, C[:, :, k])
        C[:, k, k] = R[:, k, k] = 0xFF
    return out


BAND = 32  # block size of the banded path (csrc/gj_band.cu)


def banded(bits: np.ndarray, n: int) -> np.ndarray:
    """Host restatement of band_detect_bits_kernel: (batch,) bool, True when
    every edge j -> i of the graph has |i // 32 - j // 32| <= 1."""
    bits = np.asarray(bits).view(np.uint32)
    batch = bits.shape[0]
    wpr = (n + 31) // 32
    words = bits.reshape(batch, n, wpr)
    q = np.arange(wpr)[None, :]
    outside = np.abs(q - (np.arange(n) // BAND)[:, None]) > 1
    return ~((words != 0) & outside[None]).any(axis=(1, 2))


def band_flops(n: int) -> float:
    """FP64 flop of the banded inverse of one matrix (csrc/gj_band.cu): 2 * 32^3
    per block product or block inverse; (nb - 1)(nb + 5) products (sweeps,
    diagonal, chains) and 3 nb inverses, nb = n_pad / 32."""
    nb = L.pad_to_nb(n) // BAND
    return float((nb - 1) * (nb + 5) + 3 * nb) * 2.0 * BAND**3


S0_CAP = 24  # sparse first step: edges per row / column of 256-wide step-0 blocks (csrc/gj_invert.cu S0<256>)
S0_CAP_512 = 32  # ... of the two-level path's 512-wide outer step-0 blocks (S0<512>)
DW_MIN_BATCH = 2  # dense-wide path: at least 2 matrices per sub-batch


def _off(key: str) -> bool:
    """An A-B switch the library reads from the environment, set to 0."""
    return os.environ.get(key, "1").startswith("0")


def _sparse_step(p: np.ndarray, n: int, b0: int, cap: int) -> bool:
    """At most ``cap`` edges in every row of p[b0:n, :b0] and every column of
    p[:b0, b0:n] (the step-0 blocks of the leading n x n problem)."""
    return bool(p[b0:n, :b0].sum(axis=1).max(initial=0) <= cap and p[:b0, b0:n].sum(axis=0).max(initial=0) <= cap)


def two_level(n: int, batch: int) -> bool:
    """The dense-wide matrices of this batch take the two-level path (n = 1024:
    two 512-wide outer steps, csrc/gj_invert.cu dw2_part)."""
    return L.pad_to_nb(n) == 1024 and batch >= DW_MIN_BATCH and not _off("RDB_GJ_DW2")


def dense_wide_classes(bits: np.ndarray, n: int) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Host restatement of the dense-wide path's classification
    (dw_classify_kernel, dw_s0_count / gather kernels): per matrix, whether it
    takes the dense-wide steps (not banded, every off-diagonal strip non-zero)
    and, of those, whether its first 256-wide step is sparse (at most S0_CAP
    edges in every row of block column 0 and column of block row 0; on the
    two-level path: of the leading 512 x 512 block) and whether the two-level
    path's 512-wide outer step 0 is sparse (at most S0_CAP_512).
    Returns (dense_wide, sparse_256, sparse_512) boolean masks."""
    bits = np.asarray(bits).view(np.uint32)
    batch = bits.shape[0]
    nt = L.pad_to_nb(n) // L.RDB_NB
    none = np.zeros(batch, bool)
    if (batch < DW_MIN_BATCH or nt < 4 or nt % 2 or nt > PLAN_MAX_NT or n < 2 * L.RDB_NB or _off("RDB_GJ_DW")
            or _off("RDB_GJ_BAND") or _off("RDB_GJ_SKIP")):
        return none, none, none
    band = banded(bits, n)
    pat = strip_pattern(bits, n)
    off = ~np.eye(nt, dtype=bool)
    dense = ~band & (pat[:, :, off] == 0xFF).all(axis=(1, 2))
    from .workloads import unpack_bits

    two = two_level(n, batch)
    s256, s512 = none.copy(), none.copy()
    for b in np.flatnonzero(dense) if not _off("RDB_GJ_DW_S0") else []:
        p = unpack_bits(bits[b], n)
        s256[b] = _sparse_step(p, 512 if two else n, 256, S0_CAP)
        s512[b] = two and _sparse_step(p, n, 512, S0_CAP_512)
    return dense, s256, s512


def sparse_first_step(bits: np.ndarray, n: int) -> tuple[np.ndarray, np.ndarray]:
    """(dense_wide, sparse 256-wide first step) of :func:`dense_wide_classes`."""
    dense, s256, _ = dense_wide_classes(bits, n)
    return dense, s256


def _dw_flops(p: np.ndarray, n: int, sparse0: bool) -> float:
    """Flop of one one-level dense-wide inversion of the leading n x n block:
    2 n^3, less the dense 256-wide step 0 when it is sparse (2 * 256 per edge of
    block row 0, 2 * n per edge of block column 0 instead)."""
    fl = 2.0 * n**3
    if sparse0:
        b0 = 256
        fl += 2.0 * b0 * p[:b0, b0:n].sum() + 2.0 * n * p[b0:n, :b0].sum() - (2.0 * b0 * b0 * (n - b0)
                                                                              + 2.0 * (n - b0) * b0 * n)
    return fl


def executed_flops(bits: np.ndarray, n: int) -> float:
    """FP64 flop K2 executes on this batch with the default knobs: the banded
    path for block-tridiagonal graphs, the block-sparse Gauss-Jordan plan
    (2 * 128 * 128 * 16 per k-chunk) for the others, except the dense-wide
    matrices: one-level, 2 n^3 less a sparse first step (:func:`_dw_flops`);
    two-level (n = 1024, W = 512), the two W x W inversions (the leading one
    with its own sparse first step), the outer step 0 (sparse: 2 W per edge of
    block row 0, 2 n per edge of block column 0; else its dense row panel and
    update, 2 W^3 + 2 W^2 n) and the outer step 1 (2 W^3 + 2 W^2 n)."""
    bits = np.asarray(bits)
    batch = bits.shape[0]
    nt = L.pad_to_nb(n) // L.RDB_NB
    if batch > 1 and nt <= PLAN_MAX_NT:
        band = banded(bits, n)
        dense, s256, s512 = dense_wide_classes(bits, n)
        plan = ~band & ~dense
        chunks = gj_plan_chunks(strip_pattern(bits[plan], n)).sum() if plan.any() else 0
        extra = band.sum() * band_flops(n)
        from .workloads import unpack_bits

        npad = nt * L.RDB_NB
        two = two_level(n, batch)
        for b in np.flatnonzero(dense):
            p = unpack_bits(bits[b].view(np.uint32), n)
            p = np.pad(p, ((0, npad - n), (0, npad - n)))
            if not two:
                extra += _dw_flops(p, npad, bool(s256[b]))
                continue
            w = npad // 2
            step = 2.0 * w**3 + 2.0 * w * w * npad
            outer0 = 2.0 * w * p[:w, w:].sum() + 2.0 * npad * p[w:, :w].sum() if s512[b] else step
            extra += _dw_flops(p, w, bool(s256[b])) + outer0 + 2.0 * w**3 + step
    else:
        chunks = batch * nt**3 * STRIPS
        extra = 0.0
    return float(chunks) * 2.0 * L.RDB_NB * L.RDB_NB * (L.RDB_NB // STRIPS) + extra


def _certified(rec: L.PivotInfo) -> bool:
    """No-pivot pivots all positive (nonsingular M-matrix) and above the
    reference's tolerance (linalg.py:33-38; scale = max|M| = 1 for
    M = I - gamma*A with 0 < gamma < 1)."""
    return not (rec.flags & (L.RDB_PIV_NONPOS | L.RDB_PIV_NONFINITE)) and rec.min_pivot >= PIVOT_RTOL * 1.0


def uncertified(infos: list[L.PivotInfo]) -> np.ndarray:
    """Indices of graphs whose no-pivot inverse is not certified: gamma past the
    critical gain (a non-positive pivot) or a pivot below tolerance. Their D is
    recomputed by :func:`redo_pivoted`."""
    return np.array([k for k, rec in enumerate(infos) if not _certified(rec)], dtype=np.int64)


def check_infos(infos: list[L.PivotInfo], gammas: np.ndarray, first_index: int = 0) -> None:
    """Strict form: raise ResolventSingularError for the first graph whose
    no-pivot inverse is not certified (bench.py asserts none is)."""
    for k, rec in enumerate(infos):
        if not _certified(rec):
            err = ResolventSingularError(float(gammas[k]))
            err.graph_index = first_index + k
            raise err from SingularMatrixError(
                f"graph {first_index + k}: min pivot {rec.min_pivot:.3e} (flags {rec.flags})"
            )


def redo_pivoted(bits: np.ndarray, gammas: np.ndarray, n: int, idx: np.ndarray) -> np.ndarray:
    """int32 D of the graphs ``idx`` through the drop-in single-graph path:
    the no-pivot kernel's certificate failed, so M is inverted by the
    partial-pivoting kernel, which raises ResolventSingularError exactly when
    the reference's LAPACK path does (linalg.py:32-38, resolvent.py:116-119).
    The error carries ``graph_index``."""
    from .graphs import Graph, GraphKind
    from .resolvent import resolvent, rounded_r_distance
    from .workloads import unpack_bits

    out = np.empty((len(idx), n, n), dtype=np.int32)
    for r, k in enumerate(idx):
        present = unpack_bits(np.asarray(bits)[k].view(np.uint32), n)
        g = Graph(n, np.where(present, 1.0, np.inf), GraphKind.UNWEIGHTED)
        try:
            d = rounded_r_distance(resolvent(g, float(gammas[k]), with_residual=False))
        except ResolventSingularError as err:
            err.graph_index = int(k)
            raise
        fin = np.isfinite(d)
        out[r] = np.where(fin, d, 0).astype(np.int32)
        out[r][~fin] = UNREACHABLE
    return out


class APSPBatchEngine:
    """Reusable pipeline: pinned host bits -> device -> int32 D -> pinned host.

    All kernels run back to back on one compute stream, chunk by chunk (one
    rdb_apsp_bits_batched[_d8] pipeline call per chunk); a copy
    stream moves each chunk's int32 D to pinned host memory as soon as its K3
    finishes (CUDA events), so the device->host transfer of chunk i overlaps
    the kernels of chunks i+1, i+2, ... Two D slots ping-pong; the M / work
    buffers are reused by every chunk (the compute stream orders them).
    """

    def __init__(self, n: int, max_batch: int, chunk: int = 128, d_dtype: str = "int32", use_graphs: bool = True):
        self.dev = L.device()
        self.d_dtype = D_DTYPES[d_dtype]
        self.n = n
        self.n_pad = L.pad_to_nb(n)
        self.max_batch = max_batch
        self.chunk = max(1, min(chunk, max_batch))
        wpr = (n + 31) // 32
        dev = self.dev
        # per output slot: inputs and counters, so the host->device copy of
        # batch s+1 runs while batch s computes
        self.bits = [torch.empty((max_batch, n, wpr), dtype=torch.int32, device=dev) for _ in range(2)]
        self.gammas = [torch.empty(max_batch, dtype=torch.float64, device=dev) for _ in range(2)]
        self.m = torch.empty((self.chunk, self.n_pad, self.n_pad), dtype=torch.float64, device=dev)
        self.work = torch.empty(L.lib().rdb_invert_workspace_bytes(self.n_pad, self.chunk), dtype=torch.uint8,
                                device=dev)
        self.infos = [L.pivot_info_tensor(max_batch, dev) for _ in range(2)]
        self.counters = [torch.zeros((max_batch, L.RDB_NCOUNTERS), dtype=torch.int64, device=dev)
                         for _ in range(2)]
        self.d = [torch.empty((self.chunk, n, n), dtype=self.d_dtype, device=dev) for _ in range(2)]
        self.cs = torch.cuda.Stream(device=dev)  # kernels
        self.xs = torch.cuda.Stream(device=dev)  # device -> host
        self.hs = torch.cuda.Stream(device=dev)  # host -> device
        nchunks = (max_batch + self.chunk - 1) // self.chunk
        self.uploaded = [[torch.cuda.Event() for _ in range(nchunks)] for _ in range(2)]
        self.inputs_free = [torch.cuda.Event() for _ in range(2)]
        self.computed = [torch.cuda.Event() for _ in range(2)]
        self.copied = [torch.cuda.Event() for _ in range(2)]
        self.outs = [torch.empty((max_batch, n, n), dtype=self.d_dtype).pin_memory() for _ in range(2)]
        self.info_hosts = [torch.empty(max_batch * 16, dtype=torch.uint8).pin_memory() for _ in range(2)]
        self.cnt_hosts = [torch.empty((max_batch, L.RDB_NCOUNTERS), dtype=torch.int64).pin_memory()
                          for _ in range(2)]
        self.inputs: list = [None, None]
        self.done = [torch.cuda.Event() for _ in range(2)]
        self.pending = [0, 0]
        self.dslot = 0
        self.launches = 0
        # CUDA graphs of the per-chunk pipeline call, keyed by (input slot, D slot,
        # chunk, count): captured on the second use of a key (the first runs
        # eagerly so the library's one-time setup stays outside any capture)
        self.use_graphs = use_graphs
        self.graphs: dict = {}
        self.seen: set = set()

    def pin(self, bits: np.ndarray, gammas) -> tuple[torch.Tensor, torch.Tensor]:
        """Pinned host copies of the inputs (done once, outside any timed region)."""
        bits = np.ascontiguousarray(bits)
        g = np.ascontiguousarray(np.asarray(gammas, dtype=np.float64).reshape(bits.shape[0]))
        if not np.all((g > 0) & (g < 1)):
            raise ValueError("every gamma must be in (0, 1)")
        return torch.from_numpy(bits.view(np.int32)).pin_memory(), torch.from_numpy(g).pin_memory()

    def submit(self, bits_pin: torch.Tensor, gammas_pin: torch.Tensor, slot: int = 0) -> int:
        """Enqueue the whole batch into output slot ``slot`` (0 or 1) and return
        its size; :meth:`wait` (or :meth:`finish`) collects it. Batches
        submitted to alternating slots stream back to back: the kernels of one
        overlap the device->host copy of the previous one."""
        batch = bits_pin.shape[0]
        if batch > self.max_batch:
            raise ValueError(f"batch {batch} exceeds engine capacity {self.max_batch}")
        if self.pending[slot]:
            raise RuntimeError(f"slot {slot} still holds an uncollected batch")
        self.pending[slot] = batch
        self.inputs[slot] = (bits_pin, gammas_pin)
        out, info_host, info = self.outs[slot], self.info_hosts[slot], self.infos[slot]
        bits, gam, counters = self.bits[slot], self.gammas[slot], self.counters[slot]
        cur = torch.cuda.current_stream(self.dev)
        self.cs.wait_stream(cur)
        self.xs.wait_stream(cur)
        self.hs.wait_stream(cur)
        # uploads: as soon as this slot's previous batch has finished computing
        with torch.cuda.stream(self.hs):
            self.hs.wait_event(self.inputs_free[slot])
            for idx, c0 in enumerate(range(0, batch, self.chunk)):
                cnt = min(self.chunk, batch - c0)
                bits[c0 : c0 + cnt].copy_(bits_pin[c0 : c0 + cnt], non_blocking=True)
                gam[c0 : c0 + cnt].copy_(gammas_pin[c0 : c0 + cnt], non_blocking=True)
                self.uploaded[slot][idx].record(self.hs)
        with torch.cuda.stream(self.cs):
            if self.d_dtype == torch.uint8:
                counters[:batch].zero_()
        for idx, c0 in enumerate(range(0, batch, self.chunk)):
            s = self.dslot  # D slots alternate over every chunk ever submitted
            self.dslot ^= 1
            cnt = min(self.chunk, batch - c0)
            with torch.cuda.stream(self.cs):
                self.cs.wait_event(self.uploaded[slot][idx])
                # D slot s must have drained to the host (the chunk submitted
                # two chunks earlier, in this batch or the previous one)
                self.cs.wait_event(self.copied[s])
                # K1 -> K2 -> K3 in one pipeline call (banded graphs detected
                # before K1, which then writes only their band)
                self._pipeline(slot, s, c0, cnt, bits, gam, info, counters)
                self.launches += launches_per_call(self.n, cnt)
                self.computed[s].record(self.cs)
            with torch.cuda.stream(self.xs):
                self.xs.wait_event(self.computed[s])
                out[c0 : c0 + cnt].copy_(self.d[s][:cnt], non_blocking=True)
                self.copied[s].record(self.xs)
        self.inputs_free[slot].record(self.cs)
        with torch.cuda.stream(self.xs):
            self.xs.wait_stream(self.cs)
            info_host[: batch * 16].copy_(info[: batch * 16], non_blocking=True)
            if self.d_dtype == torch.uint8:
                self.cnt_hosts[slot][:batch].copy_(counters[:batch], non_blocking=True)
            self.done[slot].record(self.xs)
        return batch

    def _pipeline(self, slot, s, c0, cnt, bits, gam, info, counters) -> None:
        """K1 -> K2 -> K3 for one chunk on the compute stream (graph replay when captured)."""
        key = (slot, s, c0, cnt)
        g = self.graphs.get(key)
        if g is not None:
            g.replay()
            return

        def call():
            apsp_call(bits[c0:], self.n, cnt, gam[c0:], self.m, self.work, info[c0 * 16 :], self.d[s],
                      counters[c0:], torch.cuda.current_stream().cuda_stream)

        if not self.use_graphs or key not in self.seen:
            self.seen.add(key)
            call()
            return
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.cs):
            call()
        self.graphs[key] = g
        g.replay()

    def wait(self, slot: int, gammas_pin: torch.Tensor, check: bool = True) -> np.ndarray:
        """Block until slot ``slot``'s batch is in host memory; its D (int32, or
        uint8 for a compact engine). A compact batch with any graph outside the
        uint8 range is returned widened to int32, those graphs recomputed."""
        batch = self.pending[slot]
        self.done[slot].synchronize()
        self.pending[slot] = 0
        out = self.outs[slot][:batch].numpy()
        bits_pin, g_pin = self.inputs[slot]
        redo = uncertified(L.read_pivot_info(self.info_hosts[slot][: batch * 16])) if check else np.zeros(0, np.int64)
        if self.d_dtype == torch.uint8:
            bad = np.nonzero(self.cnt_hosts[slot][:batch, L.RDB_CNT_D8_RANGE].numpy())[0]
            bad = np.setdiff1d(bad, redo)
            if bad.size or redo.size:
                out = decode_d8(out)
                if bad.size:
                    out[bad] = rounded_r_distance_batch(bits_pin.numpy()[bad], g_pin.numpy()[bad], self.n)
        if redo.size:
            out = out.copy() if out.base is not None else out
            out[redo] = redo_pivoted(bits_pin.numpy(), g_pin.numpy(), self.n, redo)
        return out

    def finish(self, batch: int, gammas_pin: torch.Tensor, check: bool = True) -> np.ndarray:
        return self.wait(0, gammas_pin, check)

    def run(self, bits_pin: torch.Tensor, gammas_pin: torch.Tensor, check: bool = True) -> np.ndarray:
        self.submit(bits_pin, gammas_pin, 0)
        return self.wait(0, gammas_pin, check)


def rounded_r_distance_batch(bits: np.ndarray, gammas, n: int, *, chunk: int = 64,
                             d_dtype: str = "int32") -> np.ndarray:
    """D (batch, n, n) for bit-packed unweighted graphs (host in, host out):
    int32, or uint8 (255 = unreachable; widened to int32 if a graph needs it)."""
    eng = APSPBatchEngine(n, np.asarray(bits).shape[0], chunk, d_dtype)
    b, g = eng.pin(bits, gammas)
    return eng.run(b, g).copy()


def rounded_r_distance_batch_device(bits: torch.Tensor, gammas: torch.Tensor, n: int,
                                    buf: BatchBuffers | None = None) -> torch.Tensor:
    """Device-resident variant: bits (batch, n, ceil(n/32)) int32 CUDA tensor -> int32 D on the device.

    Pivot records stay on the device in ``buf.info`` (check with
    :func:`check_infos` after a sync when needed).
    """
    batch = bits.shape[0]
    if buf is None or buf.chunk < batch or buf.n != n:
        buf = BatchBuffers.allocate(n, batch, bits.device)
    if buf.bits.data_ptr() != bits.data_ptr():
        buf.bits[:batch].copy_(bits.view(torch.int32))
    if buf.gammas.data_ptr() != gammas.data_ptr():
        buf.gammas[:batch].copy_(gammas)
    run_chunk(buf, batch)
    return buf.d[:batch]
