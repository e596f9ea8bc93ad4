"""Batched all-pairs distances for many independent unweighted graphs.

The config-2 workload: the reference's timed closure ``run_rdist``
(pkg/src/rdist/experiments.py:305-310: resolvent(g, gamma,
with_residual=False) -> r_distance -> ceil) applied to a batch of graphs
with per-graph gains, as one device pipeline per chunk: bit-packed adjacency
-> M = I - gamma*A (K1) -> batched Gauss-Jordan inverse (K2) -> int32
D = ceil(log Y / log gamma) (K3), via ``rdb_apsp_bits_batched``.

int32 D uses INT32_MAX for unreachable pairs (the reference's +inf) and 0 on
the diagonal. A graph whose inversion is not certified or is singular raises
ResolventSingularError naming the graph.

:class:`APSPBatchEngine` owns reusable device and pinned host buffers (the
serving form: host bits in, host int32 D out, copies overlapped with the
kernels on two streams); :func:`rounded_r_distance_batch` is the one-shot
convenience wrapper.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .linalg import PIVOT_RTOL, SingularMatrixError
from .resolvent import ResolventSingularError

UNREACHABLE = L.INT32_SENTINEL


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
    def allocate(cls, n: int, chunk: int, dev: torch.device) -> "BatchBuffers":
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
            d=torch.empty((chunk, n, n), dtype=torch.int32, device=dev),
            counters=torch.zeros((chunk, L.RDB_NCOUNTERS), dtype=torch.int64, device=dev),
        )

    @property
    def n_pad(self) -> int:
        return self.m.shape[-1]

    # the three stages separately (bench.py times each kernel family)
    def stage_build(self, count: int, stream: int) -> None:
        L.check(L.lib().rdb_build_m_bits(self.bits.data_ptr(), self.n, self.n_pad, count, self.gammas.data_ptr(),
                                         0.0, self.m.data_ptr(), self.n_pad, self.n_pad * self.n_pad, stream),
                "rdb_build_m_bits")

    def stage_invert(self, count: int, stream: int) -> None:
        L.check(L.lib().rdb_invert_batched(self.m.data_ptr(), self.n_pad, self.n_pad, self.n_pad * self.n_pad,
                                           count, self.work.data_ptr(), self.info.data_ptr(), stream),
                "rdb_invert_batched")

    def stage_log_ceil(self, count: int, stream: int) -> None:
        L.check(L.lib().rdb_log_ceil(self.m.data_ptr(), self.n, self.n_pad, self.n_pad * self.n_pad, count,
                                     self.gammas.data_ptr(), 0.0, None, None, self.d.data_ptr(), self.n,
                                     self.n * self.n, None, 0, self.counters.data_ptr(), stream),
                "rdb_log_ceil")


def run_chunk(buf: BatchBuffers, count: int, stream: int | None = None) -> None:
    """Launch K1 -> K2 -> K3 for the first ``count`` graphs held in ``buf``."""
    L.check(
        L.lib().rdb_apsp_bits_batched(
            buf.bits.data_ptr(), buf.n, count, buf.gammas.data_ptr(), buf.m.data_ptr(), buf.work.data_ptr(),
            buf.info.data_ptr(), buf.d.data_ptr(), buf.counters.data_ptr(),
            L.stream_handle() if stream is None else stream,
        ),
        "rdb_apsp_bits_batched",
    )


LAUNCHES_PER_CALL_FIXED = 2  # K1 + K3; K2 adds 3 per panel


def launches_per_call(n: int) -> int:
    return LAUNCHES_PER_CALL_FIXED + 3 * (L.pad_to_nb(n) // L.RDB_NB)


def check_infos(infos: list[L.PivotInfo], gammas: np.ndarray, first_index: int = 0) -> None:
    """The reference's singularity rule per graph (linalg.py:33-38; scale = max|M| = 1
    for M = I - gamma*A with 0 < gamma < 1)."""
    for k, rec in enumerate(infos):
        bad_cert = rec.flags & (L.RDB_PIV_NONPOS | L.RDB_PIV_NONFINITE)
        if bad_cert or not (rec.min_pivot >= PIVOT_RTOL * 1.0):
            g = float(gammas[k])
            err = ResolventSingularError(g)
            err.graph_index = first_index + k
            raise err from SingularMatrixError(
                f"graph {first_index + k}: min pivot {rec.min_pivot:.3e} (flags {rec.flags})"
            )


class APSPBatchEngine:
    """Reusable pipeline: pinned host bits -> device -> int32 D -> pinned host.

    All kernels run back to back on one compute stream, chunk by chunk; a copy
    stream moves each chunk's int32 D to pinned host memory as soon as its K3
    finishes (CUDA events), so the device->host transfer of chunk i overlaps
    the kernels of chunks i+1, i+2, ... Two D slots ping-pong; the M / work
    buffers are reused by every chunk (the compute stream orders them).
    """

    def __init__(self, n: int, max_batch: int, chunk: int = 128):
        self.dev = L.device()
        self.n = n
        self.n_pad = L.pad_to_nb(n)
        self.max_batch = max_batch
        self.chunk = max(1, min(chunk, max_batch))
        wpr = (n + 31) // 32
        dev = self.dev
        self.bits = torch.empty((max_batch, n, wpr), dtype=torch.int32, device=dev)
        self.gammas = torch.empty(max_batch, dtype=torch.float64, device=dev)
        self.m = torch.empty((self.chunk, self.n_pad, self.n_pad), dtype=torch.float64, device=dev)
        self.work = torch.empty(L.lib().rdb_invert_workspace_bytes(self.n_pad, self.chunk), dtype=torch.uint8,
                                device=dev)
        self.infos = [L.pivot_info_tensor(max_batch, dev) for _ in range(2)]
        self.counters = torch.zeros((max_batch, L.RDB_NCOUNTERS), dtype=torch.int64, device=dev)
        self.d = [torch.empty((self.chunk, n, n), dtype=torch.int32, device=dev) for _ in range(2)]
        self.cs = torch.cuda.Stream(device=dev)
        self.xs = torch.cuda.Stream(device=dev)
        self.computed = [torch.cuda.Event() for _ in range(2)]
        self.copied = [torch.cuda.Event() for _ in range(2)]
        self.outs = [torch.empty((max_batch, n, n), dtype=torch.int32).pin_memory() for _ in range(2)]
        self.info_hosts = [torch.empty(max_batch * 16, dtype=torch.uint8).pin_memory() for _ in range(2)]
        self.done = [torch.cuda.Event() for _ in range(2)]
        self.pending = [0, 0]
        self.launches = 0

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
        out, info_host, info = self.outs[slot], self.info_hosts[slot], self.infos[slot]
        cur = torch.cuda.current_stream(self.dev)
        self.cs.wait_stream(cur)
        self.xs.wait_stream(cur)
        lib = L.lib()
        for idx, c0 in enumerate(range(0, batch, self.chunk)):
            s = idx % 2
            cnt = min(self.chunk, batch - c0)
            with torch.cuda.stream(self.cs):
                self.bits[c0 : c0 + cnt].copy_(bits_pin[c0 : c0 + cnt], non_blocking=True)
                self.gammas[c0 : c0 + cnt].copy_(gammas_pin[c0 : c0 + cnt], non_blocking=True)
                if idx >= 2:
                    self.cs.wait_event(self.copied[s])  # slot s drained to the host
                L.check(
                    lib.rdb_apsp_bits_batched(
                        self.bits[c0].data_ptr(), self.n, cnt, self.gammas[c0:].data_ptr(), self.m.data_ptr(),
                        self.work.data_ptr(), info[c0 * 16 :].data_ptr(), self.d[s].data_ptr(),
                        self.counters[c0].data_ptr(), self.cs.cuda_stream),
                    "rdb_apsp_bits_batched",
                )
                self.launches += launches_per_call(self.n)
                self.computed[s].record(self.cs)
            with torch.cuda.stream(self.xs):
                self.xs.wait_event(self.computed[s])
                out[c0 : c0 + cnt].copy_(self.d[s][:cnt], non_blocking=True)
                self.copied[s].record(self.xs)
        with torch.cuda.stream(self.xs):
            self.xs.wait_stream(self.cs)
            info_host[: batch * 16].copy_(info[: batch * 16], non_blocking=True)
            self.done[slot].record(self.xs)
        return batch

    def wait(self, slot: int, gammas_pin: torch.Tensor, check: bool = True) -> np.ndarray:
        """Block until slot ``slot``'s batch is in host memory; its int32 D."""
        batch = self.pending[slot]
        self.done[slot].synchronize()
        self.pending[slot] = 0
        if check:
            check_infos(L.read_pivot_info(self.info_hosts[slot][: batch * 16]), gammas_pin.numpy())
        return self.outs[slot][:batch].numpy()

    def finish(self, batch: int, gammas_pin: torch.Tensor, check: bool = True) -> np.ndarray:
        return self.wait(0, gammas_pin, check)

    def run(self, bits_pin: torch.Tensor, gammas_pin: torch.Tensor, check: bool = True) -> np.ndarray:
        self.submit(bits_pin, gammas_pin, 0)
        return self.wait(0, gammas_pin, check)


def rounded_r_distance_batch(bits: np.ndarray, gammas, n: int, *, chunk: int = 64) -> np.ndarray:
    """int32 D (batch, n, n) for bit-packed unweighted graphs (host in, host out)."""
    eng = APSPBatchEngine(n, np.asarray(bits).shape[0], chunk)
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
