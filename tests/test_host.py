"""CPU tests: the C-ABI library loads and exports its header, the host-side
mirror of the reference API behaves like the reference where no GPU is
involved, and the product path refuses to run without a GPU (no fallback)."""

import ctypes
import math
import re
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2308_07403_b200 as rb
from paper_2308_07403_b200 import _lib as L
from paper_2308_07403_b200 import workloads as wl

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    text = (ROOT / "include" / "rdist_b200.h").read_text()
    return sorted(set(re.findall(r"\b(rdb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(str(L.LIB_PATH))
    names = header_functions()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name


def test_binding_table_matches_header():
    assert sorted(L.SIGNATURES) == header_functions()


def test_constants_match_header():
    text = (ROOT / "include" / "rdist_b200.h").read_text()
    defs = dict(re.findall(r"#define (RDB_[A-Z0-9_]+) (-?\d+)", text))
    for name in ("RDB_ABI_VERSION", "RDB_NB", "RDB_OK", "RDB_PIV_NONPOS", "RDB_PIV_NONFINITE", "RDB_CNT_NEGATIVE",
                 "RDB_CNT_UNDERFLOW", "RDB_CNT_D8_RANGE", "RDB_NCOUNTERS", "RDB_D8_MAX", "RDB_D8_UNREACHABLE"):
        assert getattr(L, name) == int(defs[name]), name


def test_abi_version_and_errors_without_gpu():
    lib = L.load_library()
    assert lib.rdb_abi_version() == L.RDB_ABI_VERSION
    assert lib.rdb_strerror(0) == b"ok"
    assert b"invalid" in lib.rdb_strerror(1)
    # argument validation happens before any CUDA call
    assert lib.rdb_invert(None, 128, 128, None, None, None) == 1
    assert lib.rdb_invert(ctypes.c_void_p(256), 100, 100, ctypes.c_void_p(256), ctypes.c_void_p(256), None) == 1
    assert lib.rdb_log_ceil(None, 4, 4, 0, 1, None, 0.5, None, None, None, 4, 0, None, 0, None, None) == 1
    # uint8 D needs its range counters
    assert lib.rdb_log_ceil_d8(ctypes.c_void_p(256), 4, 4, 16, 1, None, 0.5, ctypes.c_void_p(256), 4, 16, None,
                               None) == 1
    # row-block counters + dynamic tile counters + block-sparse plan (column and row strip masks,
    # per-part counts, row-panel and update tile lists, band flags and the banded-inverse
    # scratch of 4 * (n/32) 32x32 blocks per matrix) + the dense-wide path (lists, counts,
    # nested plan lists, nested / column / row counters, sparse-first-step flags and
    # lists); 256-byte aligned parts
    al = lambda x: (x + 255) // 256 * 256  # noqa: E731
    b, nt = 256, 8
    plan = (al(b * 8 * 4 + 64) + 256 + al(b * 2 * 8 * 8) + al(4 * 2 * 8 * 4) + al(b * 8 * 7 * 4)
            + al(b * 8 * 8 * 7 * 8) + al(b * 2 * 8 * 4) + al(b * 4) + al(b * 4 * 32 * 32 * 32 * 8))
    dw = (al(b * 4) + al(4 * 16 * 4) + al(4 * 16 * 4) + al(2 * b * 4) + al(4 * b * 8) + al((2 * b + 16) * 4)
          + al(b * nt * 4) + al(b * nt * 4) + 5 * al(b * 4))  # + sparse-first-step flags and lists (2 levels)
    assert lib.rdb_invert_workspace_bytes(1024, 256) == plan + dw
    assert lib.rdb_invert_batched_bits(None, 128, 128, 128 * 128, 2, None, 100, None, None, None) == 1
    assert lib.rdb_invert_workspace_bytes(0, 1) == 0


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    g = rb.Graph(2, np.array([[np.inf, 1.0], [np.inf, np.inf]]), rb.GraphKind.UNWEIGHTED)
    with pytest.raises(rb.NativeUnavailableError):
        rb.resolvent(g, 0.5)
    with pytest.raises(rb.NativeUnavailableError):
        rb.lu_invert(np.eye(3))


def test_argument_errors_before_device():
    g = rb.Graph(2, np.array([[np.inf, 1.0], [np.inf, np.inf]]), rb.GraphKind.UNWEIGHTED)
    for gamma in (0.0, 1.0, -0.2, 1.5):
        with pytest.raises(ValueError):
            rb.build_x(g, gamma)
        with pytest.raises(ValueError):
            rb.resolvent(g, gamma)
    with pytest.raises(ValueError):
        rb.lu_invert(np.ones((2, 3)))
    with pytest.raises(ValueError):
        rb.greedy_descent(g, np.zeros((2, 2)), 0, 5)


class TestScalarBounds:
    def test_delta_min(self):
        assert rb.DELTA_MIN == 5e-324
        assert rb.precision_floor(1) == rb.DELTA_MIN

    def test_boundary_at_distance_323(self):
        assert rb.precision_floor(323) < 0.1
        assert rb.precision_floor(324) >= 0.1

    def test_monotone(self):
        f = [rb.precision_floor(d) for d in (1, 10, 100, 1000, 100000)]
        assert all(a < b for a, b in zip(f, f[1:])) and f[-1] < 1.0

    def test_invalid_dmax(self):
        with pytest.raises(ValueError):
            rb.precision_floor(0)

    def test_floor_clamp_wins(self):
        assert rb.suggest_gamma(rb.GammaBounds(0.1, 0.05, 300, True), 0.01) == pytest.approx(0.5)

    def test_infeasible_raises(self):
        with pytest.raises(rb.InfeasibleGammaError):
            rb.suggest_gamma(rb.GammaBounds(0.1, 0.2, 500, False))

    def test_safety_range(self):
        with pytest.raises(ValueError):
            rb.suggest_gamma(rb.GammaBounds(0.1, 1e-5, 3, True), 1.0)

    def test_acyclic(self):
        b = rb.GammaBounds(math.inf, rb.precision_floor(1), 1, True)
        assert b.max_feasible_distance == math.inf
        assert 0 < rb.suggest_gamma(b) < 1

    def test_max_feasible_distance(self):
        b = rb.GammaBounds(0.1, rb.precision_floor(400), 400, False)
        assert b.max_feasible_distance == pytest.approx(math.log(5e-324) / math.log(0.1))


class TestGraphContract:
    def test_validation(self):
        with pytest.raises(ValueError):
            rb.Graph(2, np.array([[0.0, 1.0], [1.0, np.inf]]), rb.GraphKind.UNWEIGHTED)
        with pytest.raises(ValueError):
            rb.Graph(2, np.array([[np.inf, 2.0], [1.0, np.inf]]), rb.GraphKind.UNWEIGHTED)
        with pytest.raises(ValueError):
            rb.Graph(2, np.array([[np.inf, 1.5], [1.0, np.inf]]), rb.GraphKind.INTEGER_WEIGHTED)
        with pytest.raises(ValueError):
            rb.Graph(2, np.array([[np.inf, -1.0], [1.0, np.inf]]), rb.GraphKind.REAL_WEIGHTED)
        g = rb.Graph(2, np.array([[np.inf, 1.0], [np.inf, np.inf]]), rb.GraphKind.UNWEIGHTED)
        assert not g.weights.flags.writeable and g.num_edges == 1

    def test_edge_list_orientation(self):
        g = rb.graph_from_edge_list(rb.EdgeList(3, ((0, 2, 1.0),)), rb.GraphKind.UNWEIGHTED)
        assert g.weights[2, 0] == 1.0 and list(g.successors(0)) == [2]
        for bad in (((0, 0, 1.0),), ((0, 3, 1.0),), ((0, 1, 1.0), (0, 1, 1.0)), ((0, 1, 2.0),)):
            with pytest.raises(ValueError):
                rb.graph_from_edge_list(rb.EdgeList(3, bad), rb.GraphKind.UNWEIGHTED)

    def test_adjacency_indicator(self):
        g = rb.graph_from_edge_list(rb.EdgeList(3, ((0, 1, 1.0), (1, 2, 1.0))), rb.GraphKind.UNWEIGHTED)
        assert rb.adjacency_indicator(g).tolist() == [[0, 0, 0], [1, 0, 0], [0, 1, 0]]

    def test_resolvent_name_is_the_function(self):
        import paper_2308_07403_b200

        assert callable(paper_2308_07403_b200.resolvent)


class TestWorkloads:
    def test_chunked_bits_equal_full_draw(self):
        n, p, seed = 200, 0.05, 9
        full = wl.pack_bits(wl.er_present(n, p, seed))
        assert np.array_equal(wl.er_bits_chunked(n, p, seed, chunk_rows=37), full)

    def test_pack_roundtrip_odd_width(self):
        rng = np.random.default_rng(0)
        a = rng.random((3, 45, 45)) < 0.3
        assert np.array_equal(wl.unpack_bits(wl.pack_bits(a), 45), a)

    def test_lattice_arcs(self):
        p = wl.lattice_present(32, 0.8, 1000)
        assert not p.diagonal().any()
        # every arc joins grid neighbours
        dst, src = np.nonzero(p)
        dy = np.abs(dst // 32 - src // 32)
        dx = np.abs(dst % 32 - src % 32)
        assert ((dy + dx) == 1).all()
        frac = p.sum() / (4 * 32 * 32 - 4 * 32)
        assert 0.75 < frac < 0.85

    def test_cfg2_layout(self):
        seeds = wl.cfg2_seeds(256)
        assert seeds[0] == ("er", 2000) and seeds[128] == ("lattice", 1000)
        assert wl.cfg2_seeds(256, rank=1)[0] != seeds[0]

    def test_weighted_cfg4(self):
        g = wl.weighted_er_graph(100, 0.1, 1.0, 5.0, 3)
        fin = np.isfinite(g.weights)
        assert (g.weights[fin] >= 1.0).all() and (g.weights[fin] <= 5.0).all()
        assert g.kind is rb.GraphKind.REAL_WEIGHTED


def test_shard_targets_partition():
    from paper_2308_07403_b200.navigation import shard_targets

    for n, world in ((4096, 8), (4096, 3), (5, 8), (1, 2)):
        parts = [shard_targets(n, r, world) for r in range(world)]
        assert np.array_equal(np.concatenate(parts), np.arange(n))
    with pytest.raises(ValueError):
        shard_targets(10, 2, 2)
