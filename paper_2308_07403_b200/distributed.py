"""2D block-cyclic Gauss-Jordan inversion across GPUs (config 5: one N = 32768 matrix).

Layout: NB x NB tiles (NB = 128) dealt block-cyclically over a P_r x P_c
process grid; rank (r, c) holds global row blocks I = r, r + P_r, ... and
column blocks J = c, c + P_c, ... as one dense row-major local matrix.

Per panel k; (kr, kc) = (k mod P_r, k mod P_c):
  1. the diagonal owner (kr, kc) inverts its tile in place: D = A_kk^-1 (P1);
  2. D is broadcast along process row kr;
  3. process row kr forms its part of the row panel in place: A_kJ = D A_kJ;
  4. the row panel is broadcast down every process column (root: row kr);
  5. the old column panel A_Ik is broadcast along every process row (root: column kc);
  6. every rank updates all its tiles: A_IJ -= A_Ik A_kJ (I != k), A_Ik = -A_Ik D.
Steps 1, 3 and 6 are the same sm_100a kernels as the single-GPU inversion
(rdb_gj_panel_inverse, rdb_gemm_local on the persistent DMMA engine) and
perform the same per-tile arithmetic in the same order, so the distributed
inverse is bitwise identical to the single-GPU one. Broadcasts are NCCL
(torch.distributed) over NVLink; a grid can also be driven entirely inside
one process (VirtualGrid: every rank's tiles on one device, broadcasts as
device copies) to validate the decomposition on a single GPU.

The communication engine and the local-compute engine are parameters so the
schedule itself is tested on CPU with gloo and a test-double engine
(tests/test_distributed.py); the product engine is CudaEngine (no CPU path).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _lib as L

NB = L.RDB_NB


@dataclass(frozen=True)
class Layout:
    n: int
    pr: int
    pc: int
    nb: int = NB

    def __post_init__(self):
        if self.n % self.nb:
            raise ValueError(f"n = {self.n} must be a multiple of {self.nb}")
        if self.pr < 1 or self.pc < 1:
            raise ValueError("process grid dimensions must be >= 1")

    @property
    def nt(self) -> int:
        return self.n // self.nb

    def row_blocks(self, r: int) -> list[int]:
        return list(range(r, self.nt, self.pr))

    def col_blocks(self, c: int) -> list[int]:
        return list(range(c, self.nt, self.pc))

    def local_shape(self, r: int, c: int) -> tuple[int, int]:
        return len(self.row_blocks(r)) * self.nb, len(self.col_blocks(c)) * self.nb

    def rank(self, r: int, c: int) -> int:
        return r * self.pc + c

    def coords(self, rank: int) -> tuple[int, int]:
        return divmod(rank, self.pc)


def scatter(full: torch.Tensor, lay: Layout, r: int, c: int) -> torch.Tensor:
    """Rank (r, c)'s local matrix of a full n x n matrix (a strided gather)."""
    nb = lay.nb
    rows = torch.cat([torch.arange(I * nb, (I + 1) * nb) for I in lay.row_blocks(r)]) if lay.row_blocks(r) else torch.empty(0, dtype=torch.long)
    cols = torch.cat([torch.arange(J * nb, (J + 1) * nb) for J in lay.col_blocks(c)]) if lay.col_blocks(c) else torch.empty(0, dtype=torch.long)
    return full.index_select(0, rows.to(full.device)).index_select(1, cols.to(full.device)).contiguous()


def gather(locals_: dict[tuple[int, int], torch.Tensor], lay: Layout) -> torch.Tensor:
    """Inverse of scatter over all ranks' local matrices (tests / small n)."""
    any_t = next(iter(locals_.values()))
    full = torch.empty((lay.n, lay.n), dtype=any_t.dtype, device=any_t.device)
    nb = lay.nb
    for (r, c), loc in locals_.items():
        for li, I in enumerate(lay.row_blocks(r)):
            for lj, J in enumerate(lay.col_blocks(c)):
                full[I * nb:(I + 1) * nb, J * nb:(J + 1) * nb] = loc[li * nb:(li + 1) * nb, lj * nb:(lj + 1) * nb]
    return full


# ---------------------------------------------------------------- grids (communication)
class VirtualGrid:
    """Every rank of the grid driven by this process; broadcasts are copies."""

    def __init__(self, lay: Layout):
        self.lay = lay
        self.members = [(r, c) for r in range(lay.pr) for c in range(lay.pc)]

    def bcast_row(self, r: int, root_c: int, bufs: dict) -> None:
        src = bufs[(r, root_c)]
        for c in range(self.lay.pc):
            if c != root_c:
                bufs[(r, c)].copy_(src)

    def bcast_col(self, c: int, root_r: int, bufs: dict) -> None:
        src = bufs[(root_r, c)]
        for r in range(self.lay.pr):
            if r != root_r:
                bufs[(r, c)].copy_(src)

    def allreduce_min(self, x: float) -> float:
        return x

    def allreduce_or(self, x: int) -> int:
        return x


class TorchGrid:
    """This rank of a torch.distributed process grid (NCCL on GPUs, gloo on CPU).

    Row / column sub-communicators are created once (every rank creates every
    group, in the same order, as torch.distributed requires)."""

    def __init__(self, lay: Layout, rank: int | None = None):
        import torch.distributed as dist

        self.dist = dist
        self.lay = lay
        world = dist.get_world_size()
        if world != lay.pr * lay.pc:
            raise ValueError(f"world size {world} != grid {lay.pr} x {lay.pc}")
        self.rank = dist.get_rank() if rank is None else rank
        self.me = lay.coords(self.rank)
        self.members = [self.me]
        self.row_groups = [dist.new_group([lay.rank(r, c) for c in range(lay.pc)]) for r in range(lay.pr)]
        self.col_groups = [dist.new_group([lay.rank(r, c) for r in range(lay.pr)]) for c in range(lay.pc)]

    def bcast_row(self, r: int, root_c: int, bufs: dict) -> None:
        if self.me[0] != r or self.lay.pc == 1:
            return
        self.dist.broadcast(bufs[self.me], src=self.lay.rank(r, root_c), group=self.row_groups[r])

    def bcast_col(self, c: int, root_r: int, bufs: dict) -> None:
        if self.me[1] != c or self.lay.pr == 1:
            return
        self.dist.broadcast(bufs[self.me], src=self.lay.rank(root_r, c), group=self.col_groups[c])

    def _reduce(self, x: float, op) -> float:
        dev = torch.device("cuda", torch.cuda.current_device()) if self.dist.get_backend() == "nccl" else torch.device("cpu")
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=op)
        return float(t.item())

    def allreduce_min(self, x: float) -> float:
        return self._reduce(x, self.dist.ReduceOp.MIN)

    def allreduce_or(self, x: int) -> int:
        return int(self._reduce(float(x), self.dist.ReduceOp.MAX))


# ---------------------------------------------------------------- engines (local compute)
@dataclass
class CudaEngine:
    """Local tile operations on the sm_100a kernels (the product engine)."""

    infos: dict = field(default_factory=dict)  # coord -> (device pivot record, used)

    def panel_inverse(self, coord, block: torch.Tensor, k: int) -> None:
        rec = self.infos.get(coord)
        if rec is None:
            rec = [L.pivot_info_tensor(1, block.device), False]
            self.infos[coord] = rec
        L.check(L.lib().rdb_gj_panel_inverse(block.data_ptr(), block.stride(0), rec[0].data_ptr(), 0 if rec[1] else 1,
                                             k * NB, L.stream_handle()), "rdb_gj_panel_inverse")
        rec[1] = True

    def row_panel(self, d: torch.Tensor, rows: torch.Tensor, skip_col: int) -> None:
        n = rows.shape[1]
        L.check(L.lib().rdb_gemm_local(d.data_ptr(), d.stride(0), rows.data_ptr(), rows.stride(0), rows.data_ptr(),
                                       rows.stride(0), NB, n, NB, -1, skip_col, -1, 0, 0, L.stream_handle()),
                "rdb_gemm_local(row panel)")

    def update(self, c: torch.Tensor, colpanel: torch.Tensor, rowpanel: torch.Tensor, skip_row: int,
               store_col: int) -> None:
        m, n = c.shape
        L.check(L.lib().rdb_gemm_local(colpanel.data_ptr(), colpanel.stride(0), rowpanel.data_ptr(),
                                       rowpanel.stride(0), c.data_ptr(), c.stride(0), m, n, NB, skip_row, -1,
                                       store_col, 1, 1, L.stream_handle()), "rdb_gemm_local(update)")

    def pivot_summary(self) -> tuple[float, int]:
        minp, flags = float("inf"), 0
        for rec, used in self.infos.values():
            if used:
                p = L.read_pivot_info(rec)[0]
                minp = min(minp, p.min_pivot)
                flags |= p.flags
        return minp, flags


# ---------------------------------------------------------------- the schedule
def invert_block_cyclic(locals_: dict[tuple[int, int], torch.Tensor], grid, engine) -> tuple[float, int]:
    """In-place inverse of the block-cyclically distributed matrix.

    ``locals_`` maps each grid coordinate this process drives to its local
    matrix (row-major, NB-tile aligned). Returns (global min |pivot|, OR of the
    pivot flags) for the singularity rule / no-pivot certificate.
    """
    lay = grid.lay
    nb = lay.nb
    any_t = next(iter(locals_.values()))
    dev, dt = any_t.device, any_t.dtype
    dbuf = {co: torch.empty((nb, nb), dtype=dt, device=dev) for co in grid.members}
    rbuf = {co: torch.empty((nb, locals_[co].shape[1]), dtype=dt, device=dev) for co in grid.members}
    cbuf = {co: torch.empty((locals_[co].shape[0], nb), dtype=dt, device=dev) for co in grid.members}
    for k in range(lay.nt):
        kr, kc = k % lay.pr, k % lay.pc
        lrk, lck = k // lay.pr, k // lay.pc
        # 1. P1 on the diagonal owner, D to its row's buffers
        for co in grid.members:
            if co == (kr, kc):
                loc = locals_[co]
                blk = loc[lrk * nb:(lrk + 1) * nb, lck * nb:(lck + 1) * nb]
                engine.panel_inverse(co, blk, k)
                dbuf[co].copy_(blk)
        # 2. D along process row kr
        grid.bcast_row(kr, kc, dbuf)
        # 3. row panel in place on process row kr
        for co in grid.members:
            if co[0] == kr:
                rows = locals_[co][lrk * nb:(lrk + 1) * nb]
                engine.row_panel(dbuf[co], rows, lck if co[1] == kc else -1)
        # 4. row panel down each process column (root: process row kr)
        rp = {}
        for co in grid.members:
            rp[co] = locals_[co][lrk * nb:(lrk + 1) * nb] if co[0] == kr else rbuf[co]
        for c in sorted({co[1] for co in grid.members}):
            grid.bcast_col(c, kr, rp)
        # 5. old column panel along each process row (root: process column kc)
        for co in grid.members:
            if co[1] == kc:
                cbuf[co].copy_(locals_[co][:, lck * nb:(lck + 1) * nb])
        for r in sorted({co[0] for co in grid.members}):
            grid.bcast_row(r, kc, cbuf)
        # 6. rank-NB update of every local tile
        for co in grid.members:
            engine.update(locals_[co], cbuf[co], rp[co], lrk if co[0] == kr else -1, lck if co[1] == kc else -1)
    minp, flags = engine.pivot_summary()
    return grid.allreduce_min(minp), grid.allreduce_or(flags)
