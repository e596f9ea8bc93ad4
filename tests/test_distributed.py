"""The 2D block-cyclic inversion schedule (paper_2308_07403_b200/distributed.py)
on CPU: a single-process virtual grid and real multi-process torch.distributed
grids over gloo (world size 2 and 4), with a CPU test-double engine for the
local tile operations. The GPU engine is exercised in test_gpu_distributed.py.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_07403_b200 import distributed as D

NB = D.NB


class CpuTestEngine:
    """Reference local tile operations in float64 torch on CPU (test double)."""

    def __init__(self):
        self.minp = float("inf")

    def panel_inverse(self, coord, blk, k):
        self.minp = min(self.minp, float(torch.linalg.svdvals(blk).min()))
        blk.copy_(torch.linalg.inv(blk))

    def row_panel(self, d, rows, skip_col, max_ctas=0):
        for J in range(rows.shape[1] // NB):
            if J != skip_col:
                sl = slice(J * NB, (J + 1) * NB)
                rows[:, sl] = d @ rows[:, sl]

    def update(self, c, cp, rp, skip_row, store_col, max_ctas=0):
        for I in range(c.shape[0] // NB):
            if I == skip_row:
                continue
            rs = slice(I * NB, (I + 1) * NB)
            for J in range(c.shape[1] // NB):
                cs = slice(J * NB, (J + 1) * NB)
                prod = cp[rs] @ rp[:, cs]
                if J == store_col:
                    c[rs, cs] = -prod
                else:
                    c[rs, cs] -= prod

    def pivot_summary(self):
        return self.minp, 0


def m_matrix(n, seed):
    rng = np.random.default_rng(seed)
    a = (rng.random((n, n)) < 0.05).astype(np.float64)
    np.fill_diagonal(a, 0.0)
    return np.eye(n) - 0.02 * a


def test_layout():
    lay = D.Layout(1024, 2, 4)
    assert lay.nt == 8 and lay.row_blocks(1) == [1, 3, 5, 7] and lay.col_blocks(3) == [3, 7]
    assert lay.local_shape(0, 0) == (512, 256) and lay.rank(1, 2) == 6 and lay.coords(6) == (1, 2)
    full = torch.arange(1024 * 1024, dtype=torch.float64).reshape(1024, 1024)
    locs = {(r, c): D.scatter(full, lay, r, c) for r in range(2) for c in range(4)}
    assert torch.equal(D.gather(locs, lay), full)
    with pytest.raises(ValueError):
        D.Layout(1000, 1, 2)


@pytest.mark.parametrize("grid", [(1, 1), (1, 2), (2, 1), (2, 2), (2, 4), (3, 2)])
def test_virtual_grid_cpu(grid):
    n = 768
    m = m_matrix(n, 3)
    lay = D.Layout(n, *grid)
    full = torch.from_numpy(m)
    ys = []
    for lookahead in (False, True):
        locs = {(r, c): D.scatter(full, lay, r, c) for r in range(grid[0]) for c in range(grid[1])}
        minp, flags = D.invert_block_cyclic(locs, D.VirtualGrid(lay), CpuTestEngine(), lookahead=lookahead)
        ys.append(D.gather(locs, lay).numpy())
        np.testing.assert_allclose(ys[-1], np.linalg.inv(m), rtol=1e-12, atol=1e-15)
        assert flags == 0 and minp > 0.5
    # the look-ahead order (row / column block k+1 first, the rest after the
    # next panel) gives every tile the same products in the same order
    assert np.array_equal(ys[0], ys[1])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, grid, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lay = D.Layout(n, *grid)
        m = torch.from_numpy(m_matrix(n, 5))
        tg = D.TorchGrid(lay)
        me = tg.me
        loc = D.scatter(m, lay, *me)
        minp, flags = D.invert_block_cyclic({me: loc}, tg, CpuTestEngine())
        # collect every rank's local tiles on rank 0
        gathered = [None] * world
        dist.all_gather_object(gathered, (me, loc.numpy()))
        if rank == 0:
            locs = {tuple(co): torch.from_numpy(a) for co, a in gathered}
            y = D.gather(locs, lay).numpy()
            err = float(np.max(np.abs(y - np.linalg.inv(m.numpy())) / np.maximum(np.abs(np.linalg.inv(m.numpy())), 1e-300)))
            out.put((err, minp, flags))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("grid", [(1, 2), (2, 2)])
def test_torch_grid_gloo(grid):
    world = grid[0] * grid[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, grid, 512, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    err, minp, flags = q.get(timeout=10)
    assert err < 1e-12 and flags == 0 and minp > 0.5


def test_er_bits_rows_jump_equals_full_draw():
    # a rank draws only its own rows: PCG64 jumps reproduce gen_random_dense's stream
    from paper_2308_07403_b200 import workloads as wl

    n, p, seed = 700, 0.03, 11
    full = wl.er_bits_chunked(n, p, seed, chunk_rows=128)
    rows = np.array([3, 4, 5, 130, 131, 699])
    assert np.array_equal(wl.er_bits_rows(n, p, seed, rows), full[rows])
    assert np.array_equal(wl.er_bits_parallel(n, p, seed, procs=3, chunk_rows=200), full)
    np.testing.assert_array_equal(wl.unpack_bits(full, n), wl.er_present(n, p, seed))


@pytest.mark.parametrize("grid", [(1, 2), (2, 2), (2, 3)])
def test_local_m_from_bits_is_the_scatter_of_m(grid):
    from paper_2308_07403_b200 import workloads as wl

    n, p, gamma = 768, 0.05, 1e-2
    lay = D.Layout(n, *grid)
    present = wl.er_present(n, p, 2)
    m = torch.from_numpy(np.eye(n) - gamma * present)
    for r in range(grid[0]):
        rows = [I * NB + i for I in lay.row_blocks(r) for i in range(NB)]
        br = torch.from_numpy(wl.er_bits_rows(n, p, 2, rows).view(np.int32))
        for c in range(grid[1]):
            assert torch.equal(D.local_m_from_bits(br, lay, r, c, gamma), D.scatter(m, lay, r, c))
