"""The reference's known-answer tests, run through the CUDA path.

Mirrors /root/reference/pkg/tests/test_resolvent.py, test_linalg.py and
test_navigation.py for the functions on the hot path; every call below goes
through the C ABI into the sm_100a kernels. The independent oracle is the
CPU restatement in oracle/rdist_oracle.py.
"""

import math

import numpy as np
import pytest

import paper_2308_07403_b200 as rb
import rdist_oracle as orc
from helpers import binary_tree, chain2, dense, directed_path, empty, grid, ring3, weighted

pytestmark = pytest.mark.gpu


def truncated_series(g, gamma, tail_tol=1e-12):
    x = orc.build_x(np.asarray(g.weights), gamma)
    total = np.eye(g.n_vertices)
    term = np.eye(g.n_vertices)
    for _ in range(5000):
        term = term @ x
        total += term
        if np.abs(term).max() < tail_tol:
            break
    return total


# ------------------------------------------------------------------ build_x
class TestBuildX:
    def test_no_edge_maps_to_zero(self, cuda):
        assert np.array_equal(rb.build_x(empty(3), 0.5), np.zeros((3, 3)))

    def test_unit_weight(self, cuda):
        assert rb.build_x(chain2(), 0.1)[1, 0] == 0.1

    def test_weight_three(self, cuda):
        g = rb.graph_from_edge_list(rb.EdgeList(2, ((0, 1, 3.0),)), rb.GraphKind.INTEGER_WEIGHTED)
        assert rb.build_x(g, 0.1)[1, 0] == pytest.approx(1e-3)

    def test_unweighted_equals_gamma_times_adjacency(self, cuda):
        g = dense(20, 0.4, 1)
        assert np.array_equal(rb.build_x(g, 0.013), 0.013 * rb.adjacency_indicator(g))

    def test_weighted_matches_numpy_power(self, cuda):
        g = weighted(64, 0.3, 1.0, 9.0, 3)
        x = rb.build_x(g, 1e-3)
        ref = np.power(1e-3, np.asarray(g.weights))
        np.testing.assert_allclose(x, ref, rtol=4e-16, atol=0)

    @pytest.mark.parametrize("gamma", [0.0, 1.0, -0.2, 1.5])
    def test_gamma_out_of_range(self, gamma):
        with pytest.raises(ValueError):
            rb.build_x(chain2(), gamma)


# ------------------------------------------------------------------ resolvent
class TestResolvent:
    def test_empty_graph_gives_identity(self, cuda):
        assert np.array_equal(rb.resolvent(empty(4), 0.3).y, np.eye(4))

    def test_two_vertex_chain(self, cuda):
        res = rb.resolvent(chain2(), 0.5)
        assert np.allclose(res.y, [[1.0, 0.0], [0.5, 1.0]], atol=1e-15)
        assert not res.health.negative_entries

    def test_three_ring_matches_closed_form(self, cuda):
        p = rb.adjacency_indicator(ring3())
        res = rb.resolvent(ring3(), 0.1)
        closed = (np.eye(3) + 0.1 * p + 0.01 * (p @ p)) / (1 - 1e-3)
        assert np.abs(res.y - closed).max() < 1e-12

    @pytest.mark.parametrize("make", [lambda: grid(5), lambda: binary_tree(4), lambda: dense(30, 0.3, 2)])
    def test_series_equivalence_below_half_critical(self, cuda, make):
        g = make()
        gamma = 0.5 * rb.critical_gain(g)
        assert np.abs(rb.resolvent(g, gamma).y - truncated_series(g, gamma)).max() < 1e-9

    def test_singular_at_critical_gain(self, cuda):
        with pytest.raises(rb.ResolventSingularError) as exc:
            rb.resolvent(ring3(), 1 - 1e-16)
        assert exc.value.gamma == 1 - 1e-16
        assert isinstance(exc.value.__cause__, rb.SingularMatrixError)

    def test_residual_reported(self, cuda):
        assert rb.resolvent(grid(3), 0.1).health.inversion_residual < 1e-12

    def test_residual_skippable(self, cuda):
        assert math.isnan(rb.resolvent(grid(3), 0.1, with_residual=False).health.inversion_residual)

    def test_underflow_zero_accounting(self, cuda):
        g = binary_tree(5)
        exact = orc.bfs_apsp(np.asarray(g.weights))
        reachable = np.isfinite(exact) & ~np.eye(g.n_vertices, dtype=bool)
        assert rb.resolvent(g, 1e-45, reachable=reachable).health.underflow_zeros > 0
        assert rb.resolvent(g, 0.1, reachable=reachable).health.underflow_zeros == 0

    def test_underflow_unknown_without_mask(self, cuda):
        assert rb.resolvent(grid(3), 0.1).health.underflow_zeros is None

    def test_unhealthy_past_critical_gain(self, cuda):
        # past gamma_c the no-pivot certificate fails and the pivoted kernel runs
        g = dense(12, 0.5, 0)
        gamma = min(1.9 * rb.critical_gain(g), 0.95)
        try:
            res = rb.resolvent(g, gamma)
        except rb.ResolventSingularError:
            pytest.skip("collapsed outright")
        ref = orc.resolvent_y(np.asarray(g.weights), gamma)
        assert res.health.negative_entries == bool((ref < -1e-12).any())
        np.testing.assert_allclose(res.y, ref, rtol=1e-9, atol=1e-12)
        with pytest.raises(ValueError):
            rb.communicability(res)

    def test_result_is_frozen(self, cuda):
        res = rb.resolvent(chain2(), 0.5)
        with pytest.raises(Exception):
            res.gamma = 0.2


# ------------------------------------------------------------------ r_distance
class TestRDistance:
    def test_log_identity_exact_power(self, cuda):
        y = np.array([[1.0, 0.3**2], [0.3, 1.0]])
        r = rb.r_distance(rb.ResolventResult(y, 0.3, rb.HealthFlags(False, None, 0.0)))
        assert r[0, 1] == 2.0 and r[1, 0] == 1.0

    def test_chain_distance_one(self, cuda):
        assert rb.r_distance(rb.resolvent(chain2(), 0.5))[1, 0] == 1.0

    def test_zero_maps_to_inf(self, cuda):
        assert np.isinf(rb.r_distance(rb.resolvent(chain2(), 0.5))[0, 1])

    def test_diagonal_forced_zero(self, cuda):
        assert np.array_equal(np.diag(rb.r_distance(rb.resolvent(ring3(), 0.2))), np.zeros(3))

    def test_raw_diagonal_nonpositive_before_forcing(self, cuda):
        assert np.all(np.diag(rb.resolvent(ring3(), 0.2).y) >= 1.0)

    def test_exact_powers_many_gammas(self, cuda):
        # y == gamma^k for small k must give exactly k (the ceil is not nudged)
        for gamma in (0.3, 0.1, 0.5, 1e-2, 1e-3, 0.25, 0.7):
            for k in range(1, 8):
                y = np.array([[1.0, gamma**k], [gamma, 1.0]])
                r = rb.r_distance(rb.ResolventResult(y, gamma, rb.HealthFlags(False, None, 0.0)))
                ref = orc.r_distance(y, gamma)
                assert r[1, 0] == 1.0
                assert abs(r[0, 1] - ref[0, 1]) <= 4e-16 * k

    def test_log_accuracy_full_range(self, cuda):
        # K3's table logarithm over subnormals .. 1e300, and near 1 (no cancellation)
        rng = np.random.default_rng(11)
        e = rng.uniform(-1074, 1000, size=20000)
        y = np.exp2(e) * rng.uniform(1, 2, size=e.size)
        y = np.concatenate([y, 1 + rng.uniform(-1e-3, 1e-3, 4000), 1 - np.geomspace(1e-16, 0.3, 4000),
                            [5e-324, 1e-310, 2.2250738585072014e-308, 0.7071067811865476, 1.4142135623730951]])
        y = y[np.isfinite(y) & (y > 0) & (y != 1.0)]
        k = int(np.ceil(np.sqrt(y.size)))
        mat = np.full(k * k, 0.5)
        mat[: y.size] = y
        mat = mat.reshape(k, k)
        np.fill_diagonal(mat, 1.0)
        for gamma in (0.3, 1e-3):
            r = rb.r_distance(rb.ResolventResult(mat, gamma, rb.HealthFlags(False, None, 0.0)))
            ref = orc.r_distance(mat, gamma)
            off = ~np.eye(k, dtype=bool)
            rel = np.abs(r[off] - ref[off]) / np.abs(ref[off])
            assert rel.max() < 2e-15, rel.max()

    def test_matches_oracle_logs(self, cuda):
        rng = np.random.default_rng(3)
        y = np.exp(rng.uniform(-120, 0, size=(200, 200)))
        y[rng.random((200, 200)) < 0.05] = 0.0
        res = rb.ResolventResult(y, 1e-2, rb.HealthFlags(False, None, 0.0))
        np.testing.assert_allclose(rb.r_distance(res), orc.r_distance(y, 1e-2), rtol=1e-15, atol=0)


class TestRoundedRDistance:
    def test_grid4_matches_bfs(self, cuda):
        g = grid(4)
        got = rb.rounded_r_distance(rb.resolvent(g, 1e-3))
        assert np.array_equal(got, orc.bfs_apsp(np.asarray(g.weights)))

    def test_sentinels_pass_through(self, cuda):
        rd = rb.rounded_r_distance(rb.resolvent(chain2(), 0.5))
        assert np.isinf(rd[0, 1]) and rd[1, 0] == 1.0 and rd[0, 0] == 0.0

    def test_grid4_strict_brackets(self, cuda):
        g = grid(4)
        raw = rb.r_distance(rb.resolvent(g, 1.0 / 42))
        exact = orc.bfs_apsp(np.asarray(g.weights))
        off = ~np.eye(16, dtype=bool)
        assert np.all(raw[off] > exact[off] - 1) and np.all(raw[off] < exact[off])


# ------------------------------------------------------------------ gamma bounds
class TestCriticalGain:
    def test_complete_graph_11(self, cuda):
        assert rb.critical_gain(dense(11, 1.0, 0)) == pytest.approx(0.1, abs=1e-7)

    def test_directed_ring(self, cuda):
        assert rb.critical_gain(ring3()) == pytest.approx(1.0, abs=1e-9)

    def test_directed_path_acyclic(self, cuda):
        assert rb.critical_gain(directed_path(3)) == math.inf

    def test_suggest_gamma_paper_default(self, cuda):
        gamma = rb.suggest_gamma(rb.gamma_bounds(dense(11, 1.0, 0), 50))
        assert gamma == pytest.approx(1e-3, rel=1e-4)

    def test_bounds_feasibility(self, cuda):
        g = dense(11, 1.0, 0)
        assert rb.gamma_bounds(g, 100).feasible
        b = rb.gamma_bounds(g, 400)
        assert not b.feasible and b.max_feasible_distance < 400


# ------------------------------------------------------------------ lu_invert
class TestLuInvert:
    def test_identity(self, cuda):
        assert np.array_equal(rb.lu_invert(np.eye(4)), np.eye(4))

    def test_diagonal(self, cuda):
        assert np.array_equal(rb.lu_invert(np.diag([2.0, 4.0])), np.diag([0.5, 0.25]))

    def test_unit_upper_triangular(self, cuda):
        inv = rb.lu_invert(np.array([[1.0, -0.1], [0.0, 1.0]]))
        assert np.allclose(inv, [[1.0, 0.1], [0.0, 1.0]], atol=1e-15)

    def test_singular_raises(self, cuda):
        with pytest.raises(rb.SingularMatrixError):
            rb.lu_invert(np.array([[1.0, 2.0], [2.0, 4.0]]))

    def test_zero_matrix_raises(self, cuda):
        with pytest.raises(rb.SingularMatrixError):
            rb.lu_invert(np.zeros((3, 3)))

    def test_non_square_rejected(self):
        with pytest.raises(ValueError):
            rb.lu_invert(np.ones((2, 3)))

    def test_non_finite_rejected(self, cuda):
        with pytest.raises(ValueError):
            rb.lu_invert(np.array([[1.0, np.inf], [0.0, 1.0]]))

    @pytest.mark.parametrize("seed", range(40))
    def test_inverse_residual_random(self, cuda, seed):
        # the reference's hypothesis test (test_linalg.py:59-70) on 40 seeds;
        # these need the pivoted kernel (no M-matrix certificate)
        m = np.random.default_rng(seed).uniform(-10, 10, (5, 5)) + 20.0 * np.eye(5)
        inv = rb.lu_invert(m)
        assert np.abs(inv @ m - np.eye(5)).max() < 1e-6
        np.testing.assert_allclose(inv, orc.lu_invert(m), rtol=1e-11, atol=1e-14)

    def test_golden_generic(self, cuda, golden):
        k = golden("kat")
        np.testing.assert_allclose(rb.lu_invert(k["generic5_m"]), k["generic5_inv"], rtol=1e-12, atol=1e-15)

    @pytest.mark.parametrize("n", [1, 7, 127, 128, 129, 300, 640])
    def test_m_matrix_sizes(self, cuda, n):
        # padding path (n not a multiple of 128) and multi-panel path
        g = dense(max(n, 2), min(1.0, 8.0 / max(n, 2)), n)
        m = np.eye(g.n_vertices) - orc.build_x(np.asarray(g.weights), 0.05)
        got = rb.lu_invert(m)
        ref = orc.lu_invert(m)
        np.testing.assert_allclose(got, ref, rtol=1e-13, atol=0)


class TestSpectralRadius:
    def test_complete_graph(self, cuda):
        m = np.ones((7, 7)) - np.eye(7)
        assert rb.spectral_radius(m, tol=1e-8) == pytest.approx(6, abs=1e-6)

    def test_directed_ring(self, cuda):
        p = np.array([[0.0, 0, 1], [1, 0, 0], [0, 1, 0]])
        assert rb.spectral_radius(p) == pytest.approx(1.0, abs=1e-6)

    def test_nilpotent_path(self, cuda):
        a = np.zeros((3, 3))
        a[1, 0] = a[2, 1] = 1.0
        assert rb.spectral_radius(a) == 0.0

    def test_negative_entries_rejected(self, cuda):
        with pytest.raises(ValueError):
            rb.spectral_radius(np.array([[0.0, -1.0], [1.0, 0.0]]))

    def test_non_convergence_flagged_not_raised(self, cuda):
        res = rb.power_iteration(np.diag([1.0, 0.999]), tol=1e-30, max_iter=5)
        assert not res.converged and res.iterations == 5

    @pytest.mark.parametrize("seed", range(6))
    def test_matches_oracle(self, cuda, seed):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(2, 60))
        m = rng.random((n, n))
        m = (m + m.T) / 2
        v, c, it = orc.power_iteration(m, tol=1e-9)
        got = rb.power_iteration(m, tol=1e-9)
        assert got.value == pytest.approx(v, rel=1e-12) and got.converged == c
        assert abs(got.iterations - it) <= 1

    def test_bipartite_path_graph(self, cuda):
        a = np.zeros((3, 3))
        for i, j in [(0, 1), (1, 2)]:
            a[i, j] = a[j, i] = 1.0
        assert rb.spectral_radius(a, tol=1e-10) == pytest.approx(np.sqrt(2), abs=1e-8)


# ------------------------------------------------------------------ navigation
class TestGreedyDescent:
    def test_start_equals_goal(self, cuda):
        g = directed_path(3)
        pr = rb.greedy_descent(g, orc.bfs_apsp(np.asarray(g.weights)), 2, 2)
        assert pr.vertices == [2] and pr.steps_taken == 0 and pr.reached and pr.length == 0.0

    def test_directed_path_exact(self, cuda):
        g = directed_path(3)
        pr = rb.greedy_descent(g, orc.bfs_apsp(np.asarray(g.weights)), 0, 2)
        assert pr.vertices == [0, 1, 2] and pr.reached

    def test_grid8_resolvent_estimate_optimal_everywhere(self, cuda):
        g = grid(8)
        exact = orc.bfs_apsp(np.asarray(g.weights))
        raw = rb.r_distance(rb.resolvent(g, 0.5 * rb.critical_gain(g)))
        rng = np.random.default_rng(0)
        for _ in range(60):
            start, goal = rng.integers(0, g.n_vertices, 2)
            pr = rb.greedy_descent(g, raw, int(start), int(goal))
            assert pr.reached and pr.length == exact[goal, start]

    def test_exact_estimate_weighted_length(self, cuda):
        g = weighted(20, 0.5, 1.0, 9.0, 2)
        w = np.asarray(g.weights)
        r = orc.r_distance(orc.resolvent_y(w, 1e-6), 1e-6)
        for goal in range(0, 20, 4):
            for start in range(20):
                got = rb.greedy_descent(g, r, start, goal)
                path, length, reached, steps = orc.greedy_descent(w, r, start, goal)
                assert (got.vertices, got.length, got.reached, got.steps_taken) == (path, length, reached, steps)

    def test_unreachable_goal_stops(self, cuda):
        g = directed_path(3)
        pr = rb.greedy_descent(g, orc.bfs_apsp(np.asarray(g.weights)), 2, 0)
        assert not pr.reached and pr.vertices == [2]

    def test_all_inf_estimates_stop(self, cuda):
        pr = rb.greedy_descent(directed_path(3), np.full((3, 3), np.inf), 0, 2)
        assert not pr.reached and pr.steps_taken == 0

    def test_garbage_estimate_hits_step_cap(self, cuda):
        edges = ((0, 1, 1.0), (1, 0, 1.0), (1, 2, 1.0), (2, 1, 1.0))
        g = rb.graph_from_edge_list(rb.EdgeList(3, edges), rb.GraphKind.UNWEIGHTED)
        pr = rb.greedy_descent(g, np.zeros((3, 3)), 0, 2, max_steps=7)
        assert not pr.reached and pr.steps_taken == 7

    def test_bad_vertex_rejected(self):
        g = directed_path(3)
        with pytest.raises(ValueError):
            rb.greedy_descent(g, np.zeros((3, 3)), 0, 5)

    def test_ties_pick_lowest_index(self, cuda):
        # 0 -> {1, 2, 3} all equally good toward 4
        edges = ((0, 3, 1.0), (0, 1, 1.0), (0, 2, 1.0), (1, 4, 1.0), (2, 4, 1.0), (3, 4, 1.0))
        g = rb.graph_from_edge_list(rb.EdgeList(5, edges), rb.GraphKind.UNWEIGHTED)
        d = orc.bfs_apsp(np.asarray(g.weights))
        assert rb.greedy_descent(g, d, 0, 4).vertices == [0, 1, 4]

    def test_nan_estimate_stops(self, cuda):
        g = directed_path(3)
        d = np.zeros((3, 3))
        d[2, 1] = np.nan
        pr = rb.greedy_descent(g, d, 0, 2)
        path, length, reached, steps = orc.greedy_descent(np.asarray(g.weights), d, 0, 2)
        assert (pr.vertices, pr.reached, pr.steps_taken) == (path, reached, steps)


@pytest.mark.parametrize("n,lookahead", [(1024, "1"), (2048, "1"), (2048, "0"), (4096, "1")])
def test_wide_inversion_matches_narrow(cuda, monkeypatch, n, lookahead):
    # the NB=256 single-matrix path (default for n >= 8192), with and without
    # its look-ahead, against the NB=128 path on the same M-matrix: same
    # pivots, inverse within 1e-13 relative, identical D. Small n makes the
    # side stream the longer one (the race a missing event would expose).
    import torch

    from paper_2308_07403_b200 import _device as _d
    from paper_2308_07403_b200 import _lib as L
    from paper_2308_07403_b200 import workloads as wl

    gamma = 1e-3
    g = wl.er_graph(n, 0.02, 11)
    w = _d.graph_weights(g)
    out = {}
    monkeypatch.setenv("RDB_GJ_WIDE_LA", lookahead)
    for mode, env in (("narrow", "0"), ("wide", "256")):
        monkeypatch.setenv("RDB_GJ_WIDE_MIN", env)
        m = _d.build_m(w, n, gamma, n)
        rec = _d.invert_padded_nopivot(m)
        _, d = _d.log_ceil(m, n, gamma, want_dceil=True)
        out[mode] = (m, rec, d)
    (a, ra, da), (b, rb_, db) = out["narrow"], out["wide"]
    assert ra.flags == rb_.flags == 0 and ra.min_index == rb_.min_index
    assert abs(ra.min_pivot - rb_.min_pivot) <= 1e-15
    rel = ((a - b).abs() / a.abs().clamp_min(1e-300)).max().item()
    assert rel < 1e-13, rel
    assert torch.equal(da, db)
    assert L.lib().rdb_invert_workspace_bytes(n, 1) > 0
