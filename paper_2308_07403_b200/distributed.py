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
Steps 1-5 of panel k+1 need only row block k+1 and column block k+1 after
step k's update. Look-ahead (default on CUDA): step k's update first does the
tiles of row block k+1 and column block k+1 on the compute stream; panel
k+1's steps 1-5 then run on a communication stream (into the other of two
panel buffer sets) while the rest of step k's update runs on the compute
stream with a few SMs left free (RDB_DIST_RESERVE_SMS, default 8) for the
panel kernels and NCCL's. Every tile still receives the same products in the
same order, so the result is unchanged bit for bit.
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

import os
from contextlib import nullcontext
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
    """Local tile operations on the sm_100a kernels (the product engine);
    launched on the caller's current CUDA stream."""

    infos: dict = field(default_factory=dict)  # coord -> (device pivot record, used)

    def panel_inverse(self, coord, block: torch.Tensor, k: int) -> None:
        rec = self.infos.get(coord)
        if rec is None:
            rec = [L.pivot_info_tensor(1, block.device), False]
            self.infos[coord] = rec
        L.check(L.lib().rdb_gj_panel_inverse(block.data_ptr(), block.stride(0), rec[0].data_ptr(), 0 if rec[1] else 1,
                                             k * NB, L.stream_handle()), "rdb_gj_panel_inverse")
        rec[1] = True

    def row_panel(self, d: torch.Tensor, rows: torch.Tensor, skip_col: int, max_ctas: int = 0) -> None:
        n = rows.shape[1]
        L.check(L.lib().rdb_gemm_local(d.data_ptr(), d.stride(0), rows.data_ptr(), rows.stride(0), rows.data_ptr(),
                                       rows.stride(0), NB, n, NB, -1, skip_col, -1, 0, 0, max_ctas,
                                       L.stream_handle()),
                "rdb_gemm_local(row panel)")

    def update(self, c: torch.Tensor, colpanel: torch.Tensor, rowpanel: torch.Tensor, skip_row: int,
               store_col: int, max_ctas: int = 0) -> None:
        m, n = c.shape
        if m == 0 or n == 0:
            return
        L.check(L.lib().rdb_gemm_local(colpanel.data_ptr(), colpanel.stride(0), rowpanel.data_ptr(),
                                       rowpanel.stride(0), c.data_ptr(), c.stride(0), m, n, NB, skip_row, -1,
                                       store_col, 1, 1, max_ctas, L.stream_handle()), "rdb_gemm_local(update)")

    def pivot_summary(self) -> tuple[float, int]:
        minp, flags = float("inf"), 0
        for rec, used in self.infos.values():
            if used:
                p = L.read_pivot_info(rec)[0]
                minp = min(minp, p.min_pivot)
                flags |= p.flags
        return minp, flags


# ---------------------------------------------------------------- streams
class _Streams:
    """Compute stream (the caller's current stream) + a communication stream
    for the look-ahead panels; no-ops for CPU tensors (gloo tests)."""

    def __init__(self, device: torch.device, lookahead: bool):
        self.on = lookahead  # the split schedule (also on CPU, where it runs in program order)
        self.cuda = lookahead and device.type == "cuda"
        if self.cuda:
            self.comp = torch.cuda.current_stream(device)
            self.comm = torch.cuda.Stream(device=device)

    def comm_ctx(self):
        return torch.cuda.stream(self.comm) if self.cuda else nullcontext()

    def comm_waits_comp(self):
        if self.cuda:
            self.comm.wait_stream(self.comp)

    def comp_waits_comm(self):
        if self.cuda:
            self.comp.wait_stream(self.comm)


def reserve_sms() -> int:
    return int(os.environ.get("RDB_DIST_RESERVE_SMS", "8"))


# ---------------------------------------------------------------- the schedule
def _ranges(total: int, cut: int | None) -> list[tuple[int, int]]:
    """[0, total) without the one tile index ``cut`` (None: whole range)."""
    if cut is None:
        return [(0, total)]
    return [(a, b) for a, b in ((0, cut), (cut + 1, total)) if b > a]


def _local(idx: int, blocks_mod: int, me: int) -> int | None:
    """Local tile index of global block ``idx`` on grid coordinate ``me`` (or None)."""
    return idx // blocks_mod if idx % blocks_mod == me else None


def invert_block_cyclic(locals_: dict[tuple[int, int], torch.Tensor], grid, engine,
                        lookahead: bool = True) -> tuple[float, int]:
    """In-place inverse of the block-cyclically distributed matrix.

    ``locals_`` maps each grid coordinate this process drives to its local
    matrix (row-major, NB-tile aligned). Returns (global min |pivot|, OR of the
    pivot flags) for the singularity rule / no-pivot certificate. With
    ``lookahead`` (CUDA tensors only) panel k+1 overlaps the bulk of step k's
    update (module docstring); the result is bitwise the same either way.
    """
    lay = grid.lay
    nb = lay.nb
    any_t = next(iter(locals_.values()))
    dev, dt = any_t.device, any_t.dtype
    st = _Streams(dev, lookahead)
    nsets = 2 if st.on else 1
    dbuf = [{co: torch.empty((nb, nb), dtype=dt, device=dev) for co in grid.members} for _ in range(nsets)]
    rbuf = [{co: torch.empty((nb, locals_[co].shape[1]), dtype=dt, device=dev) for co in grid.members}
            for _ in range(nsets)]
    cbuf = [{co: torch.empty((locals_[co].shape[0], nb), dtype=dt, device=dev) for co in grid.members}
            for _ in range(nsets)]
    rest_ctas, panel_ctas = 0, 0
    if st.cuda:
        panel_ctas = reserve_sms()
        rest_ctas = max(1, torch.cuda.get_device_properties(dev).multi_processor_count - panel_ctas)

    def panels(k: int, s: int) -> dict:
        """Steps 1-5 of panel k into buffer set s; returns the row panels."""
        kr, kc = k % lay.pr, k % lay.pc
        lrk, lck = k // lay.pr, k // lay.pc
        for co in grid.members:  # 1. P1 on the diagonal owner, D to its row's buffers
            if co == (kr, kc):
                blk = locals_[co][lrk * nb:(lrk + 1) * nb, lck * nb:(lck + 1) * nb]
                engine.panel_inverse(co, blk, k)
                dbuf[s][co].copy_(blk)
        grid.bcast_row(kr, kc, dbuf[s])  # 2. D along process row kr
        for co in grid.members:  # 3. row panel in place on process row kr
            if co[0] == kr:
                rows = locals_[co][lrk * nb:(lrk + 1) * nb]
                engine.row_panel(dbuf[s][co], rows, lck if co[1] == kc else -1, max_ctas=panel_ctas)
        rp = {co: (locals_[co][lrk * nb:(lrk + 1) * nb] if co[0] == kr else rbuf[s][co]) for co in grid.members}
        for c in sorted({co[1] for co in grid.members}):  # 4. row panel down each process column
            grid.bcast_col(c, kr, rp)
        for co in grid.members:  # 5. old column panel along each process row
            if co[1] == kc:
                cbuf[s][co].copy_(locals_[co][:, lck * nb:(lck + 1) * nb])
        for r in sorted({co[0] for co in grid.members}):
            grid.bcast_row(r, kc, cbuf[s])
        return rp

    def update(co, k: int, s: int, rp: dict, rows, cols, ctas: int = 0) -> None:
        """Step k's rank-NB update of co's tiles in local tile ranges rows x cols."""
        kr, kc = k % lay.pr, k % lay.pc
        lrk, lck = k // lay.pr, k // lay.pc
        loc, cp, r_ = locals_[co], cbuf[s][co], rp[co]
        for r0, r1 in rows:
            for c0, c1 in cols:
                skip = lrk - r0 if co[0] == kr and r0 <= lrk < r1 else -1
                store = lck - c0 if co[1] == kc and c0 <= lck < c1 else -1
                if skip >= 0 and r1 - r0 == 1:
                    continue
                engine.update(loc[r0 * nb:r1 * nb, c0 * nb:c1 * nb], cp[r0 * nb:r1 * nb], r_[:, c0 * nb:c1 * nb],
                              skip, store, max_ctas=ctas)

    with st.comm_ctx():
        rp = panels(0, 0)
    st.comp_waits_comm()
    for k in range(lay.nt):
        s = k % nsets
        if not st.on or k + 1 == lay.nt:
            for co in grid.members:
                mt, ntl = locals_[co].shape[0] // nb, locals_[co].shape[1] // nb
                update(co, k, s, rp, [(0, mt)], [(0, ntl)])
            if k + 1 < lay.nt:
                rp = panels(k + 1, (k + 1) % nsets)
            continue
        # tiles of row block k+1 and column block k+1 first ...
        nxt = {}
        for co in grid.members:
            mt, ntl = locals_[co].shape[0] // nb, locals_[co].shape[1] // nb
            li1, lj1 = _local(k + 1, lay.pr, co[0]), _local(k + 1, lay.pc, co[1])
            nxt[co] = (li1, lj1)
            if li1 is not None:
                update(co, k, s, rp, [(li1, li1 + 1)], [(0, ntl)])
            if lj1 is not None:
                update(co, k, s, rp, _ranges(mt, li1), [(lj1, lj1 + 1)])
        # ... then panel k+1 on the communication stream, overlapping the rest
        st.comm_waits_comp()
        with st.comm_ctx():
            rp_next = panels(k + 1, (k + 1) % nsets)
        for co in grid.members:
            mt, ntl = locals_[co].shape[0] // nb, locals_[co].shape[1] // nb
            li1, lj1 = nxt[co]
            update(co, k, s, rp, _ranges(mt, li1), _ranges(ntl, lj1), rest_ctas)
        st.comp_waits_comm()
        rp = rp_next
    minp, flags = engine.pivot_summary()
    return grid.allreduce_min(minp), grid.allreduce_or(flags)


# ---------------------------------------------------------------- config-5 inputs and outputs per rank
def local_m_from_bits(bits_rows: torch.Tensor, lay: Layout, r: int, c: int, gamma: float,
                      chunk: int = 2048) -> torch.Tensor:
    """Rank (r, c)'s local matrix of M = I - gamma*A, built on the device from
    the bit-packed adjacency rows of its own row blocks only (``bits_rows``:
    (local rows, ceil(n/32)) int32, global rows in local order, e.g. from
    workloads.er_bits_rows): M_loc[i, j] = [gi == gj] - gamma * A[gi, gj]."""
    nb = lay.nb
    rows_g = torch.tensor([I * nb + i for I in lay.row_blocks(r) for i in range(nb)], dtype=torch.long,
                          device=bits_rows.device)
    cols_g = torch.tensor([J * nb + j for J in lay.col_blocks(c) for j in range(nb)], dtype=torch.long,
                          device=bits_rows.device)
    out = torch.empty((rows_g.numel(), cols_g.numel()), dtype=torch.float64, device=bits_rows.device)
    word, shift = cols_g >> 5, (cols_g & 31).to(torch.int32)
    for a in range(0, rows_g.numel(), chunk):
        b = min(rows_g.numel(), a + chunk)
        w = bits_rows[a:b].index_select(1, word)
        out[a:b] = ((w >> shift) & 1).to(torch.float64).mul_(-gamma)
        eq = rows_g[a:b, None] == cols_g[None, :]
        out[a:b][eq] = 1.0
    return out


def local_d_columns(y_loc: torch.Tensor, lay: Layout, r: int, c: int, gamma: float,
                    cols) -> tuple[torch.Tensor, torch.Tensor]:
    """uint8 D (255 = unreachable) of this rank's rows for the sampled global
    columns it holds: (global column indices held, D (local rows, k))."""
    nb = lay.nb
    cols = torch.as_tensor(cols, dtype=torch.long, device=y_loc.device)
    mine = cols[(cols // nb) % lay.pc == c]
    lcol = (mine // nb // lay.pc) * nb + mine % nb
    k = mine.numel()
    d = torch.empty((y_loc.shape[0], k), dtype=torch.float64, device=y_loc.device)
    if k:
        ysub = y_loc.index_select(1, lcol).contiguous()
        # row0 far outside: no forced diagonal here; fixed below for the held (row == column) pairs
        L.check(L.lib().rdb_log_ceil_block(ysub.data_ptr(), ysub.shape[0], k, k, -(1 << 40), 0, mine.data_ptr(),
                                           float(gamma), None, d.data_ptr(), None, k, None, L.stream_handle()),
                "rdb_log_ceil_block")
        held = ((mine // nb) % lay.pr) == r  # global row mine[j] is one of this rank's rows
        if bool(held.any()):
            jj = torch.nonzero(held).flatten()
            lrow = (mine[jj] // nb // lay.pr) * nb + mine[jj] % nb
            d[lrow, jj] = 0.0
    u8 = torch.full(d.shape, 255, dtype=torch.uint8, device=d.device)
    fin = torch.isfinite(d)
    u8[fin] = d[fin].to(torch.uint8)
    return mine, u8
