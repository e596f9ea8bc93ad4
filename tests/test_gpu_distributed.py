"""The distributed (2D block-cyclic) inversion with the sm_100a engine, driven
as a virtual grid on one B200: every rank's tiles on the same device, the
broadcasts as device copies. Its result must be bitwise identical to the
single-GPU inversion (same per-tile arithmetic in the same order)."""

import numpy as np
import pytest
import torch

from paper_2308_07403_b200 import _device as _d
from paper_2308_07403_b200 import _lib as L
from paper_2308_07403_b200 import distributed as D
from paper_2308_07403_b200 import workloads as wl

pytestmark = pytest.mark.gpu


def m_on_device(n, gamma, seed):
    bits = torch.from_numpy(wl.pack_bits(wl.er_present(n, 0.02, seed)).view(np.int32)).cuda()
    m = torch.empty((n, n), dtype=torch.float64, device="cuda")
    L.check(L.lib().rdb_build_m_bits(bits.data_ptr(), n, n, 1, None, gamma, m.data_ptr(), n, n * n,
                                     L.stream_handle()), "build")
    return m


@pytest.mark.parametrize("lookahead", [True, False])
@pytest.mark.parametrize("grid", [(1, 1), (1, 2), (2, 1), (2, 2), (2, 4), (3, 2)])
def test_virtual_grid_bitwise_equals_single_gpu(cuda, grid, lookahead):
    n, gamma = 1024, 1e-2
    m = m_on_device(n, gamma, 17)
    ref = m.clone()
    rec = _d.invert_padded_nopivot(ref)
    lay = D.Layout(n, *grid)
    locs = {(r, c): D.scatter(m, lay, r, c) for r in range(grid[0]) for c in range(grid[1])}
    eng = D.CudaEngine()
    minp, flags = D.invert_block_cyclic(locs, D.VirtualGrid(lay), eng, lookahead=lookahead)
    y = D.gather(locs, lay)
    torch.cuda.synchronize()
    assert torch.equal(y, ref), float((y - ref).abs().max())
    assert flags == 0 and minp == rec.min_pivot


def test_gemm_local_skip_store(cuda):
    # rdb_gemm_local semantics against torch on the same device
    torch.manual_seed(0)
    m, n, k = 384, 512, 128
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    c0 = torch.randn(m, n, dtype=torch.float64, device="cuda")
    c = c0.clone()
    L.check(L.lib().rdb_gemm_local(a.data_ptr(), k, b.data_ptr(), n, c.data_ptr(), n, m, n, k, 1, -1, 2, 1, 1, 0,
                                   L.stream_handle()), "gemm")
    exp = c0 - a @ b
    exp[:, 256:384] = -(a @ b)[:, 256:384]
    exp[128:256] = c0[128:256]
    torch.cuda.synchronize()
    torch.testing.assert_close(c, exp, rtol=1e-13, atol=1e-12)


def test_torch_grid_nccl_single_rank(cuda):
    # the product grid (TorchGrid over a real NCCL process group) on this one
    # GPU: a 1 x 1 grid, so the collectives (all-reduce of the pivot summary)
    # run through NCCL; the result must equal the single-GPU inversion bitwise
    import socket

    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        n, gamma = 512, 1e-2
        m = m_on_device(n, gamma, 5)
        ref = m.clone()
        rec = _d.invert_padded_nopivot(ref)
        lay = D.Layout(n, 1, 1)
        locs = {(0, 0): D.scatter(m, lay, 0, 0)}
        minp, flags = D.invert_block_cyclic(locs, D.TorchGrid(lay), D.CudaEngine())
        torch.cuda.synchronize()
        assert torch.equal(D.gather(locs, lay), ref)
        assert flags == 0 and minp == rec.min_pivot
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("grid", [(1, 2), (2, 2), (2, 4)])
def test_cfg5_pipeline_per_rank_virtual(cuda, grid):
    """The bench's config-5 multi-GPU leg on one device: every rank builds its
    local M from the bit rows of its own row blocks only (workloads.er_bits_rows,
    a PCG64 jump per run of rows), the grid inverts with look-ahead, each rank
    takes D of the sampled columns it holds; the assembled columns equal the
    single-GPU pipeline's (single.py) bit for bit."""
    from paper_2308_07403_b200 import single as S

    n, p, gamma, seed = 2048, 0.02, 1e-3, 4
    lay = D.Layout(n, *grid)
    locs = {}
    for r in range(grid[0]):
        rows = [I * D.NB + i for I in lay.row_blocks(r) for i in range(D.NB)]
        br = torch.from_numpy(wl.er_bits_rows(n, p, seed, rows).view(np.int32)).cuda()
        for c in range(grid[1]):
            locs[(r, c)] = D.local_m_from_bits(br, lay, r, c, gamma)
    bits = torch.from_numpy(wl.er_bits_chunked(n, p, seed).view(np.int32)).cuda()
    m = S.build_m_bits(bits, n, gamma)
    assert torch.equal(D.gather(locs, lay), m)
    minp, flags = D.invert_block_cyclic(locs, D.VirtualGrid(lay), D.CudaEngine())
    assert flags == 0
    cols = np.sort(np.random.default_rng(1).choice(n, 300, replace=False))
    S.invert_in_place(m, gamma)
    want = S.d_columns(m, n, gamma, cols)
    want_u8 = torch.where(torch.isfinite(want), want, torch.full_like(want, 255)).to(torch.uint8)
    got = torch.zeros((n, len(cols)), dtype=torch.uint8, device="cuda")
    pos = {int(cg): j for j, cg in enumerate(cols)}
    for (r, c), yl in locs.items():
        held, du = D.local_d_columns(yl, lay, r, c, gamma, cols)
        rows = torch.tensor([I * D.NB + i for I in lay.row_blocks(r) for i in range(D.NB)], device="cuda")
        for j, cg in enumerate(held.tolist()):
            got[rows, pos[cg]] = du[:, j]
    assert torch.equal(got, want_u8)
