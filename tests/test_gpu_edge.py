"""Edge cases of the batch and K3 paths (round-2 review items).

- A batched graph whose no-pivot inverse is not certified (gamma past the
  critical gain, or exactly singular) goes through the partial-pivoting path,
  as the reference's LAPACK lu_invert does (linalg.py:32-38): a nonsingular
  M gives the reference's D, a singular one raises ResolventSingularError
  naming the graph (resolvent.py:116-119).
- K3 with gamma close to 1 (1 - 1e-7): the near-integer threshold grows
  without a cap, so every element takes the exact path and D equals
  ceil(log y / log gamma) (resolvent.py:140-153) on log-uniform y.
- ResolventResult is the reference's frozen dataclass (resolvent.py:60-64).
"""

import dataclasses
import math

import numpy as np
import pytest
import torch

import paper_2308_07403_b200 as rb
import rdist_oracle as orc
from paper_2308_07403_b200 import _lib as L
from paper_2308_07403_b200 import batch as B
from paper_2308_07403_b200 import workloads as wl

pytestmark = pytest.mark.gpu


def _complete(n):
    p = np.ones((n, n), bool)
    np.fill_diagonal(p, False)
    return p


@pytest.mark.parametrize("d_dtype", ["int32", "uint8"])
def test_batch_past_critical_gain_matches_reference(cuda, d_dtype):
    n = 64  # complete digraph: rho = 63, critical gain 1/63
    presents = [_complete(n), wl.er_present(n, 0.1, 3), _complete(n), wl.er_present(n, 0.2, 4)]
    gammas = np.array([0.05, 1e-2, 0.2, 0.3])  # graphs 0, 2 (and maybe 3) past the critical gain
    bits = np.stack([wl.pack_bits(p) for p in presents])
    d = rb.rounded_r_distance_batch(bits, gammas, n, d_dtype=d_dtype)
    assert d.dtype == np.int32  # uncertified graphs widen a compact batch
    for b, (p, g) in enumerate(zip(presents, gammas)):
        ref = orc.d_to_int32(orc.run_rdist(wl.weights_from_present(p), g))
        np.testing.assert_array_equal(d[b], ref, err_msg=f"graph {b}")
    # negative entries past the critical gain: those pairs are unreachable (+inf)
    assert (d[0][~np.eye(n, dtype=bool)] == rb.UNREACHABLE).any()


def test_batch_singular_graph_raises_with_index(cuda):
    n = 64
    presents = [wl.er_present(n, 0.1, 3), _complete(n)]
    gammas = np.array([1e-2, 1.0 / 63.0])  # M = I - A/63 is singular (A 1 = 63 * 1)
    bits = np.stack([wl.pack_bits(p) for p in presents])
    with pytest.raises(rb.ResolventSingularError) as exc:
        rb.rounded_r_distance_batch(bits, gammas, n)
    assert exc.value.graph_index == 1
    assert exc.value.gamma == pytest.approx(1.0 / 63.0)
    # the reference raises on the same graph
    with pytest.raises(Exception):
        orc.run_rdist(wl.weights_from_present(presents[1]), gammas[1])


@pytest.mark.parametrize("n", [255, 256])
@pytest.mark.parametrize("gamma", [1 - 1e-7, 1 - 2e-7, 1 - 1e-6, 0.999])
def test_k3_gamma_near_one(cuda, n, gamma):
    rng = np.random.default_rng(n)
    y = np.exp(rng.uniform(math.log(1e-6), 0.0, (n, n)))
    y[: n // 4] = np.exp(rng.uniform(math.log(0.9995), 0.0, (n // 4, n)))  # R < ~5000: the refined range
    res = rb.ResolventResult(y, gamma, rb.HealthFlags(False, None, 0.0))
    with np.errstate(divide="ignore"):
        r = np.log(y) / math.log(gamma)
    np.fill_diagonal(r, 0.0)
    ref = np.ceil(r)
    np.testing.assert_array_equal(rb.rounded_r_distance(res), ref)  # fp64 D (drop-in)
    # the int32 batch K3 (n % 4 != 0 takes the generic kernel, n == 256 the lean one)
    m = torch.from_numpy(y[None]).to(cuda)
    d = torch.empty((1, n, n), dtype=torch.int32, device=cuda)
    cnt = torch.zeros((1, L.RDB_NCOUNTERS), dtype=torch.int64, device=cuda)
    gam = torch.tensor([gamma], dtype=torch.float64, device=cuda)
    B.log_ceil_call(m, n, 1, gam, d, cnt, L.stream_handle())
    big = ref > np.iinfo(np.int32).max
    got = d.cpu().numpy()[0]
    np.testing.assert_array_equal(got[~big], ref[~big].astype(np.int64))


def test_resolvent_result_is_the_reference_dataclass(cuda):
    g = wl.er_graph(40, 0.2, 1)
    res = rb.resolvent(g, 1e-2)
    assert [f.name for f in dataclasses.fields(res)] == ["y", "gamma", "health"]
    with pytest.raises(dataclasses.FrozenInstanceError):
        res.gamma = 0.5
    y = res.y  # host copy of the device inverse
    assert y.shape == (40, 40) and np.allclose(y @ (np.eye(40) - orc.build_x(np.asarray(g.weights), 1e-2)), np.eye(40))
    res2 = dataclasses.replace(res, gamma=1e-2)
    np.testing.assert_array_equal(rb.rounded_r_distance(res2), rb.rounded_r_distance(res))
    assert dataclasses.asdict(res)["health"]["inversion_residual"] == res.health.inversion_residual


def _sync_or_die(seconds, what):
    """Device synchronisation with a deadline. A kernel spinning on an in-kernel
    wait never returns and no Python-level timeout can interrupt
    cudaDeviceSynchronize, so a deadlock ends the process here (with a message)
    instead of hanging the test run."""
    import os
    import sys
    import time

    done = torch.cuda.Event()
    for st in _ALL_STREAMS:
        torch.cuda.current_stream().wait_stream(st)
    done.record()
    t0 = time.monotonic()
    while not done.query():
        if time.monotonic() - t0 > seconds:
            sys.stderr.write(f"\nDEADLOCK: {what}: the GPU work did not finish in {seconds:.0f} s\n")
            sys.stderr.flush()
            os._exit(3)
        time.sleep(0.002)
    torch.cuda.synchronize()


_ALL_STREAMS: list = []


def test_concurrent_inversions_on_three_streams_make_progress(cuda):
    """Forward progress of K2's in-kernel waits with several persistent update
    kernels in flight (gj_invert.cu: tiles by atomic ticket): two batched calls
    (each split into two sub-batch streams) and a single-matrix look-ahead
    inversion issued on three user streams at once, repeatedly; every result
    equals its serial run."""
    from paper_2308_07403_b200 import single as S

    seeds = wl.cfg2_seeds(256)
    sets = [seeds[0:32] + seeds[128:160], seeds[32:64] + seeds[160:192]]
    bufs, refs = [], []
    for pick in sets:
        bits = np.stack([wl.pack_bits(wl.cfg2_present(k, s)) for k, s in pick])
        gam = np.array([wl.cfg2_gamma(k) for k, _ in pick])
        buf = B.BatchBuffers.allocate(1024, len(pick), cuda)
        buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
        buf.gammas.copy_(torch.from_numpy(gam))
        B.run_chunk(buf, len(pick))
        torch.cuda.synchronize()
        refs.append(buf.d.clone())
        bufs.append(buf)
    n = 2048
    b2 = torch.from_numpy(wl.er_bits_chunked(n, 0.02, 9).view(np.int32)).to(cuda)
    m0 = S.build_m_bits(b2, n, 1e-3)
    m_ref = m0.clone()
    S.invert_in_place(m_ref, 1e-3)
    streams = [torch.cuda.Stream() for _ in range(3)]
    _ALL_STREAMS[:] = streams
    for _ in range(6):
        m = m0.clone()
        torch.cuda.synchronize()
        for st, buf in zip(streams[:2], bufs):
            with torch.cuda.stream(st):
                B.run_chunk(buf, buf.chunk, st.cuda_stream)
        with torch.cuda.stream(streams[2]):
            work = torch.empty(L.lib().rdb_invert_workspace_bytes(n, 1), dtype=torch.uint8, device=cuda)
            info = L.pivot_info_tensor(1, cuda)
            L.check(L.lib().rdb_invert(m.data_ptr(), n, n, work.data_ptr(), info.data_ptr(), streams[2].cuda_stream),
                    "rdb_invert")
        _sync_or_die(120.0, "concurrent inversions on three streams")
        for buf, ref in zip(bufs, refs):
            assert torch.equal(buf.d, ref)
        assert torch.equal(m, m_ref)


def test_four_concurrent_dense_batches_make_progress(cuda):
    """Four batched calls of dense ER graphs (unsplit: one stream each plus the
    shared side streams) in flight at once, so every persistent launch gets only
    a few resident CTAs and a CTA often draws consecutive tiles: the case in
    which a CTA used to spin on a dependency group whose next tile it held
    itself (dmma_engine.cuh, Tile::wait). Results equal the serial runs."""
    seeds = wl.cfg2_seeds(256)[:128]  # the ER half
    bufs, refs = [], []
    for k in range(4):
        pick = seeds[12 * k: 12 * k + 12]
        bits = np.stack([wl.pack_bits(wl.cfg2_present(kind, s)) for kind, s in pick])
        gam = np.array([wl.cfg2_gamma(kind) for kind, _ in pick])
        buf = B.BatchBuffers.allocate(1024, len(pick), cuda)
        buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
        buf.gammas.copy_(torch.from_numpy(gam))
        B.run_chunk(buf, len(pick))
        torch.cuda.synchronize()
        refs.append(buf.d.clone())
        bufs.append(buf)
    streams = [torch.cuda.Stream() for _ in range(4)]
    _ALL_STREAMS[:] = streams
    for _ in range(8):
        for buf in bufs:
            buf.d.fill_(-1)
        torch.cuda.synchronize()
        for st, buf in zip(streams, bufs):
            with torch.cuda.stream(st):
                B.run_chunk(buf, buf.chunk, st.cuda_stream)
        _sync_or_die(120.0, "four concurrent dense batches")
        for buf, ref in zip(bufs, refs):
            assert torch.equal(buf.d, ref)


def test_progress_beside_a_gpu_hog(cuda):
    """The config-2 style batch (split into two sub-batch streams) while another
    stream keeps the SMs busy with large FP32 GEMMs: the persistent launches
    then get their SMs a few at a time, in no particular order, and must still
    finish with the same D."""
    seeds = wl.cfg2_seeds(256)
    pick = seeds[0:40] + seeds[128:168]
    bits = np.stack([wl.pack_bits(wl.cfg2_present(kind, s)) for kind, s in pick])
    gam = np.array([wl.cfg2_gamma(kind) for kind, _ in pick])
    buf = B.BatchBuffers.allocate(1024, len(pick), cuda)
    buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
    buf.gammas.copy_(torch.from_numpy(gam))
    B.run_chunk(buf, len(pick))
    torch.cuda.synchronize()
    ref = buf.d.clone()
    hog_a = torch.randn((6144, 6144), device=cuda)
    hog_b = torch.randn((6144, 6144), device=cuda)
    hog_c = torch.empty_like(hog_a)
    hog, work = torch.cuda.Stream(), torch.cuda.Stream()
    _ALL_STREAMS[:] = [hog, work]
    for _ in range(5):
        buf.d.fill_(-1)
        torch.cuda.synchronize()
        with torch.cuda.stream(hog):
            for _ in range(12):
                torch.matmul(hog_a, hog_b, out=hog_c)
        with torch.cuda.stream(work):
            B.run_chunk(buf, buf.chunk, work.cuda_stream)
        _sync_or_die(120.0, "batched inversion beside a GEMM hog")
        assert torch.equal(buf.d, ref)


@pytest.mark.parametrize("n,count", [(512, 72), (1024, 24), (1536, 24)])  # 72: the two-stream split
def test_mixed_batch_dense_wide_plan_and_band_paths(cuda, monkeypatch, n, count):
    """One batched call whose matrices take all three inversion paths at once:
    fully dense ER graphs (dense 256-wide steps), graphs with zero strips
    (block-sparse NB = 128 plan) and block-tridiagonal graphs (banded inverse),
    interleaved so both sub-batch streams hold a mix; D equal to the oracle and
    to the same call with the dense-wide path switched off (RDB_GJ_DW=0)."""
    rng = np.random.default_rng(n)
    i, j = np.indices((n, n))
    presents = []
    for k in range(count):
        kind = k % 3
        if kind == 0:
            q = rng.random((n, n)) < 0.03  # dense: every strip has edges
        elif kind == 1:
            q = np.zeros((n, n), bool)  # two components: zero off-diagonal blocks
            h = n // 2
            q[:h, :h] = rng.random((h, h)) < 0.03
            q[h:, h:] = rng.random((n - h, n - h)) < 0.03
        else:
            q = (np.abs(i - j) <= 20) & (np.abs(i // 32 - j // 32) <= 1) & (rng.random((n, n)) < 0.3)
        np.fill_diagonal(q, False)
        presents.append(q)
    gam = np.array([1e-2, 1e-2, 0.05] * (count // 3))
    bits = np.stack([wl.pack_bits(q) for q in presents])
    d_dw = rb.rounded_r_distance_batch(bits, gam, n)
    monkeypatch.setenv("RDB_GJ_DW", "0")
    d_plan = rb.rounded_r_distance_batch(bits, gam, n)
    np.testing.assert_array_equal(d_dw, d_plan)
    for b in range(0, len(presents), 5):
        ref = orc.d_to_int32(orc.run_rdist(wl.weights_from_present(presents[b]), gam[b]))
        np.testing.assert_array_equal(d_dw[b], ref, err_msg=f"graph {b}")


@pytest.mark.parametrize("n,p", [(512, 0.03), (1024, 0.02), (1536, 0.012)])
def test_sparse_first_step_matches_dense_steps(cuda, monkeypatch, n, p):
    """The sparse first step(s) of the dense-wide path (edge lists snapshotted,
    half-warp-per-column row panel, warp-per-row update; two levels at
    n = 1024) against the same matrices through dense tiles only
    (RDB_GJ_DW_S0=0): the inverse agrees to rounding (the sums run in another
    order), D is identical, and the APSP pipeline (M from the bits, every edge
    -gamma) gives bitwise the inverse of the generic entry point (edge values
    read from M). One graph exceeds the per-row edge cap and keeps the dense
    step."""
    from paper_2308_07403_b200 import batch as B

    rng = np.random.default_rng(n)
    count = 12
    presents = []
    for k in range(count):
        q = rng.random((n, n)) < p
        if k == 5:
            q[n - 7, :200] = True  # 200 edges into block 0 from one row: over the cap
        np.fill_diagonal(q, False)
        presents.append(q)
    bits = np.stack([wl.pack_bits(q) for q in presents])
    gam = np.full(count, 1e-2)
    dev = torch.device("cuda")
    sh = torch.cuda.current_stream().cuda_stream
    out = {}
    for mode in ("default", "dense"):
        monkeypatch.delenv("RDB_GJ_DW_S0", raising=False)
        if mode == "dense":
            monkeypatch.setenv("RDB_GJ_DW_S0", "0")
        buf = B.BatchBuffers.allocate(n, count, dev)
        buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
        buf.gammas.copy_(torch.from_numpy(gam))
        buf.stage_build(count, sh)
        buf.stage_invert(count, sh)
        torch.cuda.synchronize()
        y = buf.m.clone()
        B.run_chunk(buf, count, sh)
        torch.cuda.synchronize()
        out[mode] = (y, buf.m.clone(), buf.d.clone())
        del buf
    y_s, y_pipe, d_s = out["default"]
    y_d, _, d_d = out["dense"]
    if not torch.equal(y_s, y_pipe):  # constant-value lists == values gathered from M
        msg = []
        for b in range(count):
            dd = y_s[b] != y_pipe[b]
            if dd.any():
                idx = dd.nonzero()
                msg.append(f"graph {b}: {int(dd.sum())} entries, rows {int(idx[:, 0].min())}..{int(idx[:, 0].max())}, "
                           f"cols {int(idx[:, 1].min())}..{int(idx[:, 1].max())}")
        raise AssertionError("pipeline Y != generic Y: " + "; ".join(msg))
    assert torch.equal(d_s, d_d)
    rel = ((y_s - y_d).abs() / y_d.abs().clamp_min(1e-300)).max().item()
    assert rel < 1e-12, rel
    ref = orc.d_to_int32(orc.run_rdist(wl.weights_from_present(presents[5]), 1e-2))
    got = rb.rounded_r_distance_batch(bits[5:6], gam[5:6], n)[0]
    np.testing.assert_array_equal(got, ref)
