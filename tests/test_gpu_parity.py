"""Config-level parity of the CUDA path against the reference (golden
fixtures produced by the reference itself) and the CPU oracle.

Bars (BASELINE.json north_star): D and next hops bit-exact; R within 1e-9
relative where R <= 50 (checked far tighter here where the oracle is run on
the same inputs).
"""

import numpy as np
import pytest
import torch

import paper_2308_07403_b200 as rb
import rdist_oracle as orc
from helpers import u8_to_d
from paper_2308_07403_b200 import workloads as wl

pytestmark = pytest.mark.gpu

R_RTOL = 1e-9  # north_star tolerance for real-valued R


def int32_to_d(d32):
    d = d32.astype(np.float64)
    d[d32 == rb.UNREACHABLE] = np.inf
    return d


def test_cfg1_full(cuda, golden):
    f = golden("cfg1")
    g = wl.er_graph(512, 0.05, int(f["seed"]))
    res = rb.resolvent(g, 1e-3)
    d = rb.rounded_r_distance(res)
    np.testing.assert_array_equal(d, u8_to_d(f["d"]))
    r = rb.r_distance(res)
    np.testing.assert_allclose(r, f["r"], rtol=1e-13, atol=0)
    assert res.health.inversion_residual < 1e-12 and not res.health.negative_entries
    assert rb.critical_gain(g) == pytest.approx(float(f["critical_gain"]), rel=1e-12)


@pytest.mark.parametrize("name", ["cfg2_er_2000", "cfg2_lattice_1000", "cfg2_lattice_1001", "cfg2_lattice_1004"])
def test_cfg2_golden_batch_api(cuda, golden, name):
    f = golden(name)
    kind, seed, gamma = str(f["kind"]), int(f["seed"]), float(f["gamma"])
    bits = wl.pack_bits(wl.cfg2_present(kind, seed))[None]
    d32 = rb.rounded_r_distance_batch(bits, [gamma], 1024)
    np.testing.assert_array_equal(int32_to_d(d32[0]), u8_to_d(f["d"]))


def test_cfg2_golden_drop_in_api(cuda, golden):
    # the same graphs through the reference-shaped per-graph API
    for name in ("cfg2_er_2000", "cfg2_lattice_1004"):
        f = golden(name)
        kind, seed, gamma = str(f["kind"]), int(f["seed"]), float(f["gamma"])
        g = rb.Graph(1024, wl.weights_from_present(wl.cfg2_present(kind, seed)), rb.GraphKind.UNWEIGHTED)
        d = rb.rounded_r_distance(rb.resolvent(g, gamma, with_residual=False))
        np.testing.assert_array_equal(d, u8_to_d(f["d"]))


def test_cfg2_batch_mixed_gammas_vs_oracle(cuda):
    # a 16-graph slice of the config-2 batch (ER + lattice, mixed gains)
    seeds = wl.cfg2_seeds(256)
    pick = seeds[120:136]
    present = [wl.cfg2_present(k, s) for k, s in pick]
    bits = np.stack([wl.pack_bits(p) for p in present])
    gammas = np.array([wl.cfg2_gamma(k) for k, _ in pick])
    d32 = rb.rounded_r_distance_batch(bits, gammas, 1024, chunk=5)
    for b, (p, gm) in enumerate(zip(present, gammas)):
        ref = orc.run_rdist(wl.weights_from_present(p), gm)
        np.testing.assert_array_equal(int32_to_d(d32[b]), ref, err_msg=f"graph {pick[b]}")


def test_cfg2_full_batch_properties(cuda):
    # all 256 graphs, device-resident path; size-independent properties:
    # zero diagonal, D == 1 exactly on edges, D >= 2 elsewhere, sentinel
    # exactly where the graph has no path (zero pattern of Y = reachability)
    bits, gammas, seeds = wl.cfg2_batch(256)
    dev_bits = torch.from_numpy(bits.view(np.int32)).cuda()
    d = rb.rounded_r_distance_batch_device(dev_bits, torch.from_numpy(gammas).cuda(), 1024).cpu().numpy()
    host = rb.rounded_r_distance_batch(bits[:8], gammas[:8], 1024)
    np.testing.assert_array_equal(d[:8], host)
    for b in range(0, 256, 17):
        present = wl.unpack_bits(bits[b], 1024)
        db = d[b]
        assert (np.diagonal(db) == 0).all()
        assert (db[present] == 1).all()
        off = ~present & ~np.eye(1024, dtype=bool)
        assert (db[off] >= 2).all()
        reach = np.isfinite(orc.bfs_apsp(wl.weights_from_present(present)))
        assert np.array_equal(db != rb.UNREACHABLE, reach), seeds[b]


def test_cfg4_small_golden(cuda, golden):
    f = golden("cfg4_small")
    n = int(f["n"])
    g = wl.weighted_er_graph(n, 0.1, 1.0, 5.0, int(f["seed"]))
    r = rb.r_distance(rb.resolvent(g, 1e-3, with_residual=False))
    np.testing.assert_allclose(r, f["r"], rtol=1e-13, atol=0)
    nxt = rb.next_hop_table(g, r)
    np.testing.assert_array_equal(nxt, f["next"].astype(np.int32))
    for s, t, length, reached, steps, nv in f["paths"]:
        pr = rb.greedy_descent(g, f["r"], int(s), int(t))
        assert (pr.length, int(pr.reached), pr.steps_taken, len(pr.vertices)) == (length, int(reached), int(steps), int(nv))


def test_cfg4_full_sampled_targets(cuda):
    c = wl.CFG4
    g = wl.weighted_er_graph(c["n"], c["p"], c["w_lo"], c["w_hi"], 42)
    w = np.asarray(g.weights)
    r = rb.r_distance(rb.resolvent(g, c["gamma"], with_residual=False))
    r_ref = orc.r_distance(orc.resolvent_y(w, c["gamma"]), c["gamma"])
    fin = np.isfinite(r_ref) & (r_ref <= 50)
    assert np.array_equal(np.isfinite(r), np.isfinite(r_ref))
    rel = np.abs(r[fin] - r_ref[fin]) / np.maximum(np.abs(r_ref[fin]), 1e-300)
    assert rel.max() < R_RTOL and rel.max() < 1e-13
    targets = np.random.default_rng(1).choice(c["n"], 256, replace=False)
    got = rb.next_hop_table(g, r_ref, targets)
    ref = orc.next_hop_table(w, r_ref, targets)
    np.testing.assert_array_equal(got, ref)
    # and from the GPU's own R (ties/gaps are far above the R error)
    np.testing.assert_array_equal(rb.next_hop_table(g, r, targets), ref)


def test_cfg3_full(cuda):
    c = wl.CFG3
    g = wl.er_graph(c["n"], c["p"], 0)
    w = np.asarray(g.weights)
    d = rb.rounded_r_distance(rb.resolvent(g, c["gamma"], with_residual=False))
    ref = orc.run_rdist(w, c["gamma"])
    np.testing.assert_array_equal(d, ref)
    assert set(np.unique(d[~np.eye(c["n"], dtype=bool)])) <= {1.0, 2.0}


# ---- compact uint8 D (serving form): identical D, 255 = unreachable ----------
def test_cfg2_uint8_matches_int32_full_batch(cuda):
    from paper_2308_07403_b200 import batch as B

    bits, gammas, _ = wl.cfg2_batch(256)
    dev = torch.device("cuda")
    out = {}
    for dt in ("int32", "uint8"):
        buf = B.BatchBuffers.allocate(1024, 256, dev, d_dtype=dt)
        buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
        buf.gammas.copy_(torch.from_numpy(gammas))
        buf.counters.zero_()
        B.run_chunk(buf, 256)
        torch.cuda.synchronize()
        if dt == "uint8":
            assert B.d8_range_errors(buf.counters).size == 0
        out[dt] = buf.d.cpu().numpy()
    np.testing.assert_array_equal(B.decode_d8(out["uint8"]), out["int32"])
    assert out["uint8"].max() == rb.UNREACHABLE_D8 or (out["int32"] != rb.UNREACHABLE).all()


def test_cfg2_uint8_engine_golden(cuda, golden):
    names = ["cfg2_er_2000", "cfg2_lattice_1000", "cfg2_lattice_1001", "cfg2_lattice_1004"]
    fs = [golden(nm) for nm in names]
    bits = np.stack([wl.pack_bits(wl.cfg2_present(str(f["kind"]), int(f["seed"]))) for f in fs])
    gammas = [float(f["gamma"]) for f in fs]
    d8 = rb.rounded_r_distance_batch(bits, gammas, 1024, chunk=3, d_dtype="uint8")
    assert d8.dtype == np.uint8
    for b, f in enumerate(fs):
        np.testing.assert_array_equal(int32_to_d(rb.decode_d8(d8[b])), u8_to_d(f["d"]))


def test_uint8_range_overflow_widens_to_int32(cuda):
    # a directed path 0 -> 1 -> ... -> 299: D reaches 299 > 254, so the compact
    # engine must flag the graph on the device and hand back exact int32 D
    n = 300
    present = np.zeros((n, n), dtype=bool)
    present[np.arange(1, n), np.arange(n - 1)] = True  # [i][j]: edge j -> i
    bits = wl.pack_bits(present)[None]
    ref = rb.rounded_r_distance_batch(bits, [0.1], n)
    out = rb.rounded_r_distance_batch(np.concatenate([bits, bits]), [0.1, 0.1], n, d_dtype="uint8")
    assert out.dtype == np.int32
    np.testing.assert_array_equal(out[0], ref[0])
    np.testing.assert_array_equal(out[1], ref[0])
    assert ref[0].max() == rb.UNREACHABLE and ref[0][n - 1, 0] == n - 1


def test_cfg4_table_sharded_by_targets(cuda):
    # config 4 sharded by target rows: the ranks' row blocks
    # concatenate to the full table (computed here rank by rank on one GPU)
    from paper_2308_07403_b200.navigation import next_hop_table_shard

    g = wl.weighted_er_graph(512, 0.1, 1.0, 5.0, 3)
    r = rb.r_distance(rb.resolvent(g, 1e-3, with_residual=False))
    full = rb.next_hop_table(g, r)
    parts = [next_hop_table_shard(g, r, k, 3) for k in range(3)]
    assert np.array_equal(np.concatenate([p[0] for p in parts]), np.arange(512))
    np.testing.assert_array_equal(np.concatenate([p[1] for p in parts]), full)


@pytest.mark.parametrize("n", [1, 2, 31, 33, 100, 129, 300])
@pytest.mark.parametrize("d_dtype", ["int32", "uint8"])
def test_batch_ragged_sizes_vs_oracle(cuda, n, d_dtype):
    # sizes off every kernel granule (32-bit words, 128-wide panels, 128-column
    # K3 blocks), mixed gains, a chunk size that splits the batch unevenly
    rng = np.random.default_rng(n)
    present = [(rng.random((n, n)) < min(0.9, 3.0 / max(n, 1))) & ~np.eye(n, dtype=bool) for _ in range(5)]
    bits = np.stack([wl.pack_bits(p) for p in present])
    gammas = np.array([0.01, 0.05, 0.1, 0.02, 0.003])
    d = rb.rounded_r_distance_batch(bits, gammas, n, chunk=2, d_dtype=d_dtype)
    if d.dtype == np.uint8:
        d = rb.decode_d8(d)
    for b in range(5):
        ref = orc.run_rdist(wl.weights_from_present(present[b]), gammas[b])
        np.testing.assert_array_equal(int32_to_d(d[b]), ref, err_msg=f"n={n} graph {b}")


def test_bits_from_edge_list(cuda):
    # wire format -> device bit-packed adjacency (rdb_edges_to_bits) == host packing
    present = wl.er_present(300, 0.05, 4)
    g = rb.Graph(300, wl.weights_from_present(present), rb.GraphKind.UNWEIGHTED)
    bits = rb.bits_from_edge_list(rb.edge_list_from_graph(g)).cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(bits, wl.pack_bits(present))
    with pytest.raises(ValueError):
        rb.bits_from_edge_list(rb.EdgeList(3, ((0, 1, 2.0),)))
    with pytest.raises(ValueError):
        rb.bits_from_edge_list(rb.EdgeList(3, ((0, 3, 1.0),)))


@pytest.mark.parametrize("seed", [0, 1])
def test_next_hop_pruned_equals_unpruned_with_ties(cuda, monkeypatch, seed):
    # integer weights and integer "distances" make exact score ties everywhere:
    # the weight-sorted, bound-pruned scan must pick the same (lowest-index)
    # successor as the ascending scan and the oracle restatement
    from paper_2308_07403_b200 import _device as _d

    n = 700
    rng = np.random.default_rng(seed)
    present = (rng.random((n, n)) < 0.05) & ~np.eye(n, dtype=bool)
    w = np.where(present, rng.integers(1, 4, (n, n)).astype(np.float64), np.inf)
    dist = rng.integers(0, 6, (n, n)).astype(np.float64)
    dist[rng.random((n, n)) < 0.05] = np.inf
    wd = torch.from_numpy(w).cuda()
    dd = torch.from_numpy(dist).cuda()
    tg = torch.arange(n, dtype=torch.int32, device="cuda")
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("RDB_NEXT_HOP_PRUNED", mode)
        out[mode] = _d.next_hop(wd, dd, tg).cpu().numpy()
    np.testing.assert_array_equal(out["1"], out["0"])
    ref = orc.next_hop_table(w, dist, np.arange(0, n, 7))
    np.testing.assert_array_equal(out["1"][::7], ref)


def test_batch_split_and_dynamic_are_bitwise_neutral(cuda, monkeypatch):
    # sub-batch streams and dynamic tile scheduling change only which SM does
    # which tile: every matrix's inverse is bitwise the same
    from paper_2308_07403_b200 import batch as B

    bits, gammas, _ = wl.cfg2_batch(256)
    bits, gammas = bits[96:224], gammas[96:224]  # 64 ER + 64 lattice graphs
    dev = torch.device("cuda")
    out = {}
    # (the banded path for the lattices has its own rounding order: off here,
    # compared separately in test_banded_path_matches_gauss_jordan)
    monkeypatch.setenv("RDB_GJ_BAND", "0")
    for name, env in (("default", {}), ("no_split", {"RDB_GJ_SPLIT_MIN": "0"}),
                      ("dynamic", {"RDB_GJ_DYNAMIC": "1"}), ("four", {"RDB_GJ_SPLIT_PARTS": "4"}),
                      ("dense", {"RDB_GJ_SKIP": "0"})):
        for k in ("RDB_GJ_SPLIT_MIN", "RDB_GJ_DYNAMIC", "RDB_GJ_SPLIT_PARTS", "RDB_GJ_SKIP"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        buf = B.BatchBuffers.allocate(1024, 128, dev)
        buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
        buf.gammas.copy_(torch.from_numpy(gammas))
        buf.stage_build(128, torch.cuda.current_stream().cuda_stream)
        buf.stage_invert(128, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        out[name] = buf.m.clone()
        del buf
    # the generic entry point finds the same block pattern by scanning M
    for k in ("RDB_GJ_SPLIT_MIN", "RDB_GJ_DYNAMIC", "RDB_GJ_SPLIT_PARTS", "RDB_GJ_SKIP"):
        monkeypatch.delenv(k, raising=False)
    buf = B.BatchBuffers.allocate(1024, 128, dev)
    buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
    buf.gammas.copy_(torch.from_numpy(gammas))
    buf.stage_build(128, torch.cuda.current_stream().cuda_stream)
    buf.stage_invert_generic(128, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    out["generic"] = buf.m.clone()
    for name in ("no_split", "dynamic", "four", "dense", "generic"):
        assert torch.equal(out[name], out["default"]), name


def _structured_presents(n, rng):
    """Graphs whose NB x NB block pattern stays partly zero through the
    elimination: disconnected blocks, a band, a forward-only DAG, a single
    long cycle, an empty graph, a hub, and a random sparse graph."""
    out = []
    # two components (vertex halves), each ER: off-diagonal blocks stay zero
    p = np.zeros((n, n), bool)
    h = n // 2
    p[:h, :h] = rng.random((h, h)) < 0.05
    p[h:, h:] = rng.random((n - h, n - h)) < 0.05
    out.append(p)
    # band of half-width 5 with random arcs
    i, j = np.indices((n, n))
    out.append((np.abs(i - j) <= 5) & (rng.random((n, n)) < 0.7))
    # forward DAG (edge j -> i only for i > j): strictly lower triangular
    out.append((i > j) & (rng.random((n, n)) < 0.01))
    # one directed cycle through up to 600 vertices in a random order (with
    # gamma = 0.5, y = 2^-d stays a normal double)
    perm = rng.permutation(n)[:600]
    c = np.zeros((n, n), bool)
    c[perm[1:], perm[:-1]] = True
    c[perm[0], perm[-1]] = True
    out.append(c)
    out.append(np.zeros((n, n), bool))
    hub = np.zeros((n, n), bool)  # vertex n-1 -> everyone, everyone -> vertex 0
    hub[:, n - 1] = True
    hub[0, :] = True
    out.append(hub)
    out.append(rng.random((n, n)) < 2.0 / n)
    for q in out:
        np.fill_diagonal(q, False)
    return out


@pytest.mark.parametrize("n", [300, 1024])
def test_block_sparse_schedule_structured_graphs(cuda, monkeypatch, n):
    # the block-sparse plan skips tiles of structurally zero blocks: D must
    # equal the oracle and the dense schedule on graphs that exercise it
    rng = np.random.default_rng(n)
    presents = _structured_presents(n, rng) + [wl.lattice_present(int(np.sqrt(n)), 0.8, 5)] * (n == 1024)
    # per-graph gains below each graph's critical gain that keep gamma^D_max a
    # normal double (components, band, DAG, cycle: y = 2^-d exactly, empty,
    # hub, sparse random, lattice)
    gam = np.array([1e-3, 0.1, 0.05, 0.5, 0.5, 0.1, 0.1, 0.1][: len(presents)])
    bits = np.stack([wl.pack_bits(q) for q in presents])
    outs = {}
    monkeypatch.setenv("RDB_GJ_BAND", "0")
    for mode in ("1", "0"):
        monkeypatch.setenv("RDB_GJ_SKIP", mode)
        outs[mode] = rb.rounded_r_distance_batch(bits, gam, n)
    np.testing.assert_array_equal(outs["1"], outs["0"])
    # the banded path (band, empty graph and lattice are block tridiagonal)
    monkeypatch.setenv("RDB_GJ_SKIP", "1")
    monkeypatch.setenv("RDB_GJ_BAND", "1")
    outs["band"] = rb.rounded_r_distance_batch(bits, gam, n)
    for b, q in enumerate(presents):
        w = wl.weights_from_present(q)
        r = orc.r_distance(orc.resolvent_y(w, gam[b]), gam[b])
        ref = orc.d_to_int32(np.ceil(r))
        # DAGs, cycles and sparse random graphs have pairs joined by a single
        # path: y == gamma^d up to rounding, so R sits within ulps of an integer
        # and ceil(R) is d or d + 1 depending on the last bit (the reference's
        # own knife edge; K3 returns d for y == gamma^d).
        # Exact everywhere else; on those entries D is one of the two.
        with np.errstate(invalid="ignore"):
            knife = np.isfinite(r) & (np.abs(r - np.round(r)) < 1e-9) & (r != 0)
        k = np.round(r[knife]).astype(np.int64)
        for mode in ("1", "band"):
            got = outs[mode][b]
            np.testing.assert_array_equal(got[~knife], ref[~knife], err_msg=f"graph {b} {mode}")
            assert np.isin(got[knife] - k, [0, 1]).all(), f"graph {b} {mode}"
        got = outs["1"][b]
        if b == 3:  # the gamma = 0.5 cycle: y == 2^-d exactly, so D is the hop count
            np.testing.assert_array_equal(got, orc.d_to_int32(orc.bfs_apsp(w)))


def _banded_presents(n, rng):
    """Block-tridiagonal patterns (every edge within |i/32 - j/32| <= 1) and
    near misses: a directed lattice of side 32 (n = 1024), a random band of
    half-width 32, the widest edges the band allows (i = 32q + 31 <-> j =
    32(q + 1) + 31), a path, and one graph with a single edge outside the band."""
    i, j = np.indices((n, n))
    out = []
    if n == 1024:
        out.append(wl.lattice_present(32, 0.8, 17))
    out.append((np.abs(i - j) <= 32) & (np.abs(i // 32 - j // 32) <= 1) & (rng.random((n, n)) < 0.2))
    wide = (np.abs(i // 32 - j // 32) <= 1) & (rng.random((n, n)) < 0.05)
    wide[31::32, :] |= (np.abs(i[31::32] // 32 - j[31::32] // 32) == 1) & (j[31::32] % 32 == 0)
    out.append(wide)
    path = np.zeros((n, n), bool)
    path[np.arange(1, n), np.arange(n - 1)] = True
    out.append(path)
    miss = (np.abs(i - j) <= 3) & (rng.random((n, n)) < 0.5)
    miss[n - 1, 0] = True  # one edge outside the band: Gauss-Jordan
    out.append(miss)
    for q in out:
        np.fill_diagonal(q, False)
    return out


@pytest.mark.parametrize("n", [300, 1024])
def test_banded_path_matches_gauss_jordan(cuda, monkeypatch, n):
    # K2b (gj_band.cu) against Gauss-Jordan on the same matrices: inverse
    # within 1e-12 componentwise, identical D, pivot records agree, and D
    # equal to the oracle away from the reference's own knife edges
    from paper_2308_07403_b200 import batch as B
    from paper_2308_07403_b200 import _lib as L

    rng = np.random.default_rng(n + 1)
    presents = _banded_presents(n, rng)
    gam = np.array([0.1, 0.02, 0.05, 0.6, 0.1][-len(presents):])  # 0.6^1023 stays a normal double
    bits = np.stack([wl.pack_bits(q) for q in presents])
    cnt = len(presents)
    dev = torch.device("cuda")
    ys, infos = {}, {}
    for mode in ("0", "1"):
        monkeypatch.setenv("RDB_GJ_BAND", mode)
        buf = B.BatchBuffers.allocate(n, cnt, dev)
        buf.bits.copy_(torch.from_numpy(bits.view(np.int32)))
        buf.gammas.copy_(torch.from_numpy(gam))
        sh = torch.cuda.current_stream().cuda_stream
        buf.stage_build(cnt, sh)
        buf.stage_invert(cnt, sh)
        torch.cuda.synchronize()
        ys[mode] = buf.m.cpu().numpy()[:, :n, :n]
        infos[mode] = L.read_pivot_info(buf.info)
        del buf
    for b in range(cnt):
        ya, yb = ys["0"][b], ys["1"][b]
        assert np.array_equal(ya == 0, yb == 0), b
        nz = ya != 0
        assert np.max(np.abs(yb[nz] - ya[nz]) / np.abs(ya[nz])) < 1e-12, b
        ia, ib = infos["0"][b], infos["1"][b]
        assert ia.flags == ib.flags == 0, b
        assert abs(ia.min_pivot - ib.min_pivot) <= 1e-14 * ia.min_pivot, b
    outs = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("RDB_GJ_BAND", mode)
        outs[mode] = rb.rounded_r_distance_batch(bits, gam, n)
    for b, q in enumerate(presents):
        w = wl.weights_from_present(q)
        r = orc.r_distance(orc.resolvent_y(w, gam[b]), gam[b])
        ref = orc.d_to_int32(np.ceil(r))
        with np.errstate(invalid="ignore"):
            knife = np.isfinite(r) & (np.abs(r - np.round(r)) < 1e-9) & (r != 0)
        for mode in ("0", "1"):
            np.testing.assert_array_equal(outs[mode][b][~knife], ref[~knife], err_msg=f"graph {b} band={mode}")


@pytest.mark.parametrize("d_dtype", ["uint8", "int32"])
def test_lean_k3_adversarial_values(cuda, d_dtype):
    """The batch K3 (lean kernel: FP32 MUFU estimate, exact FP64 path within its
    error bound of an integer) on values placed around every gamma^k: relative
    offsets from 1e-16 to 1e-3 either side (the estimate's threshold lies in
    that range for every gamma below), log-uniform values, zeros, negatives and
    subnormals. D must equal ceil(np.log(y) / log(gamma)) (resolvent.py:140-153)
    except at the reference's own knife edge (|R - k| < 1e-9, DESIGN.md
    "Exactness"), where k or k + 1 is accepted."""
    from paper_2308_07403_b200 import _lib as L
    from paper_2308_07403_b200 import batch as B

    n = 256
    gammas = np.array([1e-2, 0.1, 1e-5, 0.5, 0.9, 1e-3])
    rng = np.random.default_rng(5)
    deltas = np.array([0.0, 1e-16, 3e-16, 1e-13, 1e-10, 1e-8, 3e-8, 1e-7, 2e-7, 4e-7, 1e-6, 2e-6, 5e-6, 1e-5,
                       3e-5, 1e-4, 1e-3])
    deltas = np.concatenate([deltas, -deltas[1:]])
    ys = []
    for g in gammas:
        kmax = int(min(200, np.floor(np.log(1e-300) / np.log(g))))
        ks = np.arange(1, kmax + 1)
        base = np.power(g, ks.astype(np.float64))
        near = (base[:, None] * (1.0 + deltas[None, :])).ravel()
        near = near[(near > 0) & (near < 1)]
        lo = np.log(max(g ** min(kmax, 150), 1e-300))
        rnd = np.exp(rng.uniform(lo, 0.0, n * n))
        special = [0.0, -1e-13, -0.5] + ([1e-310, 4.9e-324] if g < 0.05 else [])  # D <= 254 for uint8
        y = np.concatenate([near, special, rnd])[: n * n]
        y = rng.permutation(np.resize(y, n * n)) if y.size < n * n else rng.permutation(y)
        ys.append(y.reshape(n, n))
    Y = np.stack(ys)
    m = torch.from_numpy(Y).to(cuda)
    gam = torch.from_numpy(gammas).to(cuda)
    dt = torch.uint8 if d_dtype == "uint8" else torch.int32
    d = torch.empty((len(gammas), n, n), dtype=dt, device=cuda)
    counters = torch.zeros((len(gammas), L.RDB_NCOUNTERS), dtype=torch.int64, device=cuda)
    B.log_ceil_call(m, n, len(gammas), gam, d, counters, L.stream_handle())
    got = d.cpu().numpy()
    got = B.decode_d8(got) if d_dtype == "uint8" else got
    cnt = counters.cpu().numpy()
    for b, g in enumerate(gammas):
        y = Y[b]
        with np.errstate(divide="ignore", invalid="ignore"):
            r = np.where(y > 0, np.log(np.where(y > 0, y, 1.0)) / np.log(g), np.inf)
        np.fill_diagonal(r, 0.0)
        ref = orc.d_to_int32(np.ceil(r))
        rf = np.where(np.isfinite(r), r, 0.0)
        knife = np.isfinite(r) & (np.abs(rf - np.round(rf)) < 1e-9) & (r != 0)
        assert knife.sum() < 0.05 * n * n
        np.testing.assert_array_equal(got[b][~knife], ref[~knife], err_msg=f"gamma {g}")
        k = np.round(r[knife]).astype(np.int64)
        assert np.isin(got[b][knife] - k, [0, 1]).all(), f"gamma {g}"
        assert cnt[b, L.RDB_CNT_NEGATIVE] == int((y < -1e-12).sum())
        if d_dtype == "uint8":
            assert cnt[b, L.RDB_CNT_D8_RANGE] == 0
