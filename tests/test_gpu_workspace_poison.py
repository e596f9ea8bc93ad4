"""The batched pipeline must not read anything it has not written itself.

`compute-sanitizer --tool initcheck` is closed on this GPU pool, so this is the
repository's own initcheck for K2's workspace (row-block counters, ticket
counters, block-sparse plan, dense-wide lists and counts, sparse-first-step
lists, banded scratch): every buffer the caller hands over uninitialised — the
workspace, M, D, the pivot records — is filled with a poison pattern before the
call, for every schedule the A/B switches select, through both entry points
(rdb_apsp_bits_batched from the bits, and K1 + rdb_invert_batched + K3), split
and unsplit. D must equal, bitwise, the D of the default schedule on clean
buffers (which tests/test_gpu_full_parity.py pins to the reference's digests).

It found one such read: the two-level dense-wide path took the inner level's
list count from a slot only the sparse-first-step split wrote, so
RDB_GJ_DW_S0=0 ran with whatever the allocator had left there.

Also here, for the same reason (no sanitizer on this pool): the bench step
replayed into NaN-filled buffers is bitwise deterministic (racecheck), guard
bands around every buffer stay intact, and an electric fence — every buffer in
its own virtual-memory mapping between unmapped address ranges, flush against
the end and the start (tests/fence_run.py, in a subprocess) — shows that no
kernel reads or writes outside what it is given (memcheck). RDB_TEST_POISON /
RDB_TEST_FENCE (tests/conftest.py) apply the first and the last to every
torch.empty allocation of the whole GPU suite.
"""

import numpy as np
import pytest
import torch

from paper_2308_07403_b200 import batch as B
from paper_2308_07403_b200 import workloads as wl

pytestmark = pytest.mark.gpu

MODES = [
    {},
    {"RDB_GJ_DW_S0": "0"},
    {"RDB_GJ_DW_SYNTH": "0"},
    {"RDB_GJ_DW2": "0"},
    {"RDB_GJ_DW2": "0", "RDB_GJ_DW_S0": "0"},
    {"RDB_GJ_DW": "0"},
    {"RDB_GJ_DW_LA": "0"},
    {"RDB_GJ_DW_HELPER": "0"},
    {"RDB_GJ_BAND": "0"},
    {"RDB_GJ_SKIP": "0"},
    {"RDB_GJ_DYNAMIC": "0"},
    {"RDB_GJ_SPLIT_MIN": "0"},
]
SWITCHES = sorted({k for m in MODES for k in m})


def _poison(buf, byte):
    for t in (buf.work, buf.m, buf.d, buf.info):
        t.view(torch.uint8).fill_(byte)
    buf.counters.zero_()  # (the caller's contract for the uint8 range counters)


def _run(buf, bits, gam, count, entry, sh):
    buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
    buf.gammas.copy_(torch.from_numpy(gam))
    if entry == "pipeline":
        B.run_chunk(buf, count, sh)
    else:
        buf.stage_build(count, sh)
        (buf.stage_invert if entry == "bits" else buf.stage_invert_generic)(count, sh)
        buf.stage_log_ceil(count, sh)
    torch.cuda.synchronize()
    return buf.d.clone()


@pytest.mark.parametrize("count", [12, 72])  # one stream / two sub-batch streams
def test_poisoned_buffers_every_schedule(cuda, monkeypatch, count):
    bits, gam, _ = wl.cfg2_batch(count)  # half ER (dense-wide, two levels), half lattices (banded)
    n = wl.CFG2["n"]
    dev = torch.device("cuda")
    sh = torch.cuda.current_stream().cuda_stream
    for k in SWITCHES:
        monkeypatch.delenv(k, raising=False)
    buf = B.BatchBuffers.allocate(n, count, dev)
    _poison(buf, 0)
    ref = _run(buf, bits, gam, count, "pipeline", sh)
    del buf
    bad = []
    for mode in MODES:
        for k in SWITCHES:
            monkeypatch.delenv(k, raising=False)
        for k, v in mode.items():
            monkeypatch.setenv(k, v)
        for entry in ("pipeline", "bits", "generic"):
            for byte in (0xFF, 0x01, 0x5A):  # ints -1 / 16843009 / 1515870810; doubles NaN / tiny / 3e125
                buf = B.BatchBuffers.allocate(n, count, dev)
                _poison(buf, byte)
                try:
                    d = _run(buf, bits, gam, count, entry, sh)
                except Exception as exc:
                    raise AssertionError(f"{mode} {entry} poison {byte:#x}: {exc}") from exc
                if not torch.equal(d, ref):
                    wrong = (d != ref).flatten(1).any(1).nonzero().flatten().tolist()
                    bad.append((mode, entry, hex(byte), wrong[:8]))
                del buf, d
    assert not bad, bad


def _m_matrix(n, seed, dev):
    p = wl.er_present(n, min(1.0, 12.0 / n), seed)
    m = np.eye(n) - 0.03 * p
    return torch.from_numpy(m).to(dev)


@pytest.mark.parametrize("n", [128, 640, 2048, 8192])  # one panel / look-ahead path / wide 256-step path
def test_poisoned_workspace_single_matrix(cuda, n):
    """rdb_invert (single matrix: NB = 128 look-ahead, wide path with its R / C
    scratches) on a poisoned workspace and pivot record equals the run on a
    zeroed one, bitwise."""
    from paper_2308_07403_b200 import _lib as L

    dev = torch.device("cuda")
    a0 = _m_matrix(n, n, dev)
    outs = []
    for byte in (0x00, 0xFF, 0x5A):
        a = a0.clone()
        work = torch.empty(L.lib().rdb_invert_workspace_bytes(n, 1), dtype=torch.uint8, device=dev).fill_(byte)
        info = L.pivot_info_tensor(1, dev).fill_(byte)
        L.check(L.lib().rdb_invert(a.data_ptr(), n, n, work.data_ptr(), info.data_ptr(), L.stream_handle()),
                "rdb_invert")
        torch.cuda.synchronize()
        rec = L.read_pivot_info(info)[0]
        outs.append((a, rec.min_pivot, rec.min_index, rec.flags))
    for a, mp, mi, fl in outs[1:]:
        assert torch.equal(a, outs[0][0])
        assert (mp, mi, fl) == outs[0][1:]
    assert outs[0][3] == 0


@pytest.mark.parametrize("n", [5, 300, 1100])
def test_poisoned_workspace_pivoted(cuda, n):
    """rdb_invert_pivoted (blocked partial pivoting) on a poisoned workspace."""
    from paper_2308_07403_b200 import _lib as L

    dev = torch.device("cuda")
    a0 = torch.from_numpy(np.random.default_rng(n).uniform(-1, 1, (n, n))).to(dev)
    outs = []
    for byte in (0x00, 0xFF, 0x5A):
        a = a0.clone()
        work = torch.empty(L.lib().rdb_invert_pivoted_workspace_bytes(n), dtype=torch.uint8, device=dev).fill_(byte)
        info = L.pivot_info_tensor(1, dev).fill_(byte)
        L.check(L.lib().rdb_invert_pivoted(a.data_ptr(), n, n, work.data_ptr(), info.data_ptr(), L.stream_handle()),
                "rdb_invert_pivoted")
        torch.cuda.synchronize()
        rec = L.read_pivot_info(info)[0]
        outs.append((a, rec.min_pivot, rec.min_index, rec.flags))
    for a, mp, mi, fl in outs[1:]:
        assert torch.equal(a, outs[0][0])
        assert (mp, mi, fl) == outs[0][1:]
    ref = np.linalg.inv(a0.cpu().numpy())
    np.testing.assert_allclose(outs[0][0].cpu().numpy(), ref, rtol=1e-8, atol=1e-9)


def test_bench_step_is_deterministic(cuda):
    """The config-2 bench step (256 graphs, two sub-batch streams, side
    streams, ticketed tiles, in-kernel waits) replayed 12 times, eagerly and
    from the captured CUDA graph, gives bitwise the same inverse and D every
    time: a missing dependency between the streams' kernels or a tile reading
    an operand another tile is overwriting would show up as a differing run
    (racecheck is closed on this pool with the other sanitizer tools)."""
    bits, gam, _ = wl.cfg2_batch(256)
    dev = torch.device("cuda")
    sh = torch.cuda.current_stream().cuda_stream
    buf = B.BatchBuffers.allocate(wl.CFG2["n"], 256, dev, d_dtype="uint8")
    buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
    buf.gammas.copy_(torch.from_numpy(gam))
    B.run_chunk(buf, 256, sh)
    torch.cuda.synchronize()
    y0, d0 = buf.m.clone(), buf.d.clone()
    pipe = B.CapturedPipeline(buf, 256)
    for it in range(12):
        buf.m.fill_(float("nan"))
        buf.d.fill_(77)
        if it % 2:
            pipe.replay()
        else:
            B.run_chunk(buf, 256, sh)
        torch.cuda.synchronize()
        assert torch.equal(buf.d, d0), it
        assert torch.equal(buf.m.view(torch.int64), y0.view(torch.int64)), it


def _carve(arena, off, nbytes, guard):
    """[guard | buffer | guard] at `off` in the arena; returns (buffer view, next offset)."""
    start = off + guard
    return arena[start: start + nbytes], (start + nbytes + guard + 255) // 256 * 256


@pytest.mark.parametrize("count,d_dtype", [(12, "int32"), (72, "uint8")])
def test_no_write_outside_the_buffers(cuda, count, d_dtype):
    """Every buffer of the batched pipeline (bits, gammas, M, workspace, pivot
    records, D, counters) carved out of one arena with 1 MiB guard bands of a
    known byte on both sides: after the call all guards are intact (no kernel
    writes outside what it was given) and D equals the run on ordinary
    allocations."""
    bits, gam, _ = wl.cfg2_batch(count)
    n = wl.CFG2["n"]
    dev = torch.device("cuda")
    sh = torch.cuda.current_stream().cuda_stream
    ref_buf = B.BatchBuffers.allocate(n, count, dev, d_dtype=d_dtype)
    ref = _run(ref_buf, bits, gam, count, "pipeline", sh)
    guard = 1 << 20
    sizes = {k: getattr(ref_buf, k).numel() * getattr(ref_buf, k).element_size()
             for k in ("bits", "gammas", "m", "work", "info", "d", "counters")}
    total = sum((v + 2 * guard + 255) // 256 * 256 for v in sizes.values()) + 256
    arena = torch.full((total,), 0xA5, dtype=torch.uint8, device=dev)
    views, off = {}, 0
    for k, nbytes in sizes.items():
        views[k], off = _carve(arena, off, nbytes, guard)
    like = {k: getattr(ref_buf, k) for k in sizes}
    buf = B.BatchBuffers(n=n, chunk=count, **{k: views[k].view(like[k].dtype).view(like[k].shape) for k in sizes})
    buf.counters.zero_()
    got = _run(buf, bits, gam, count, "pipeline", sh)
    assert torch.equal(got, ref)
    for k in sizes:  # wipe the buffers themselves; what is left must be all guard
        views[k].fill_(0xA5)
    assert bool((arena == 0xA5).all()), "a kernel wrote into a guard band"


@pytest.mark.parametrize("args", [("selftest",), ("12", "uint8"), ("72", "int32")])
def test_electric_fence(cuda, args):
    """tests/fence_run.py in a subprocess (a fault kills the CUDA context): every
    buffer in its own virtual-memory mapping between unmapped address ranges,
    flush against the end and then the start; `selftest` checks that an
    overread really faults."""
    import subprocess
    import sys
    from pathlib import Path

    script = Path(__file__).resolve().parent / "fence_run.py"
    proc = subprocess.run([sys.executable, str(script), *args], capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, (proc.stdout[-1500:], proc.stderr[-1500:])
