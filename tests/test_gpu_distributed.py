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


@pytest.mark.parametrize("grid", [(1, 2), (2, 1), (2, 2), (2, 4), (3, 2)])
def test_virtual_grid_bitwise_equals_single_gpu(cuda, grid):
    n, gamma = 1024, 1e-2
    m = m_on_device(n, gamma, 17)
    ref = m.clone()
    rec = _d.invert_padded_nopivot(ref)
    lay = D.Layout(n, *grid)
    locs = {(r, c): D.scatter(m, lay, r, c) for r in range(grid[0]) for c in range(grid[1])}
    eng = D.CudaEngine()
    minp, flags = D.invert_block_cyclic(locs, D.VirtualGrid(lay), eng)
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
    L.check(L.lib().rdb_gemm_local(a.data_ptr(), k, b.data_ptr(), n, c.data_ptr(), n, m, n, k, 1, -1, 2, 1, 1,
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
