"""Pin the CPU oracle against outputs of the reference itself (tests/golden).

The fixtures were produced by running the unmodified reference package
(tests/golden/make_golden.py); the oracle must reproduce them. CPU only.
"""

import hashlib
import math

import numpy as np
import pytest

import rdist_oracle as orc
from paper_2308_07403_b200 import workloads as wl


def whash(w):
    return hashlib.sha256(np.ascontiguousarray(w, dtype=np.float64).tobytes()).hexdigest()[:16]


def u8_to_d(u8):
    d = u8.astype(np.float64)
    d[u8 == 255] = np.inf
    return d


def test_kat_closed_forms(golden):
    k = golden("kat")
    assert np.array_equal(orc.resolvent_y(k["chain2_w"], 0.5), k["chain2_y"])
    assert np.allclose(k["chain2_y"], [[1.0, 0.0], [0.5, 1.0]], atol=1e-15)
    assert np.array_equal(orc.r_distance(orc.resolvent_y(k["chain2_w"], 0.5), 0.5), k["chain2_r"])
    assert np.array_equal(orc.resolvent_y(k["ring3_w"], 0.1), k["ring3_y_0p1"])
    assert np.array_equal(orc.rounded_r_distance(orc.resolvent_y(k["grid4_w"], 1e-3), 1e-3), k["grid4_d_1em3"])
    assert np.array_equal(k["grid4_d_1em3"], k["grid4_bfs"])
    assert np.array_equal(orc.bfs_apsp(k["grid4_w"]), k["grid4_bfs"])
    y = np.array([[1.0, 0.3**2], [0.3, 1.0]])
    r = orc.r_distance(y, 0.3)
    assert np.array_equal(r, k["exact_power_r"]) and r[0, 1] == 2.0 and r[1, 0] == 1.0
    assert np.array_equal(orc.lu_invert(k["generic5_m"]), k["generic5_inv"])
    rho, conv, _ = orc.power_iteration(np.ones((7, 7)) - np.eye(7), tol=1e-8)
    assert rho == float(k["complete7_rho"]) and conv


def test_cfg1_full(golden):
    f = golden("cfg1")
    w = wl.er_graph(512, 0.05, int(f["seed"])).weights
    assert whash(w) == str(f["w_hash"])
    y = orc.resolvent_y(w, 1e-3)
    r = orc.r_distance(y, 1e-3)
    np.testing.assert_array_equal(np.ceil(r), u8_to_d(f["d"]))
    np.testing.assert_allclose(r, f["r"], rtol=1e-13, atol=0)
    np.testing.assert_array_equal(orc.bfs_apsp(w), u8_to_d(f["d"]))
    rho, _, it = orc.power_iteration(np.isfinite(w).astype(np.float64))
    assert rho == pytest.approx(float(f["rho"]), rel=1e-14) and it == int(f["rho_iters"])
    m = np.eye(512) - orc.build_x(w, 1e-3)
    assert orc.residual(m, y) == pytest.approx(float(f["residual"]), rel=0.5, abs=1e-16)


@pytest.mark.parametrize("name", ["cfg2_er_2000", "cfg2_lattice_1000", "cfg2_lattice_1001", "cfg2_lattice_1004"])
def test_cfg2_samples(golden, name):
    f = golden(name)
    kind, seed, gamma = str(f["kind"]), int(f["seed"]), float(f["gamma"])
    present = wl.cfg2_present(kind, seed)
    w = wl.weights_from_present(present)
    assert whash(w) == str(f["w_hash"])
    d = orc.run_rdist(w, gamma)
    np.testing.assert_array_equal(d, u8_to_d(f["d"]))
    # the bit-packed device input format round-trips the pattern
    assert np.array_equal(wl.unpack_bits(wl.pack_bits(present), 1024), present)


def test_cfg4_small_next_hops(golden):
    f = golden("cfg4_small")
    n = int(f["n"])
    g = wl.weighted_er_graph(n, 0.1, 1.0, 5.0, int(f["seed"]))
    assert whash(g.weights) == str(f["w_hash"])
    r = orc.r_distance(orc.resolvent_y(np.asarray(g.weights), 1e-3), 1e-3)
    np.testing.assert_allclose(r, f["r"], rtol=1e-12)
    nxt = orc.next_hop_table(np.asarray(g.weights), f["r"])
    np.testing.assert_array_equal(nxt, f["next"].astype(np.int32))
    for s, t, length, reached, steps, nv in f["paths"]:
        path, ln, ok, st = orc.greedy_descent(np.asarray(g.weights), f["r"], int(s), int(t))
        assert (ln, int(ok), st, len(path)) == (length, int(reached), int(steps), int(nv))


def test_int32_format():
    d = np.array([[0.0, np.inf], [3.0, 0.0]])
    assert orc.d_to_int32(d).tolist() == [[0, 2147483647], [3, 0]]
    assert math.isinf(u8_to_d(np.array([255], dtype=np.uint8))[0])


# ---- gamma-sweep accuracy (navigation.py:77-134) and BFS, pinned to the reference
SWEEP_FIXTURES = ["sweep_grid_64", "sweep_tree_63", "sweep_hanoi_81", "sweep_dense_80", "sweep_power_law_100"]


@pytest.mark.parametrize("name", SWEEP_FIXTURES)
def test_oracle_accuracy_and_bfs_vs_reference(golden, name):
    from paper_2308_07403_b200 import workloads as wl

    f = golden(name)
    n = int(f["n"])
    w = wl.weights_from_present(wl.unpack_bits(f["bits"], n))
    assert whash(w) == str(f["w_hash"])  # the stored pattern is the reference's graph
    np.testing.assert_array_equal(orc.bfs_apsp(w), f["exact"])
    raw, exact = f["acc_raw"], f["exact"]
    assert orc.global_accuracy(np.ceil(raw), exact) == float(f["acc_global_rounded"])
    assert orc.local_accuracy(w, raw, exact) == float(f["acc_local_raw"])
    assert orc.local_accuracy(w, np.ceil(raw), exact) == float(f["acc_local_rounded"])
