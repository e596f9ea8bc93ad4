"""K10 Floyd-Warshall (csrc/floyd.cu) against the reference's loop
(oracles.py:44-50, restated in oracle/rdist_oracle.floyd_warshall): bit for
bit on real weights (the blocked kernel replays each step's row / column as
the classic loop reads them), integer weights and unweighted graphs (equal
to BFS), ragged sizes and unreachable pairs."""

import numpy as np
import pytest

import paper_2308_07403_b200 as rb
import rdist_oracle as orc
from helpers import dense, grid, weighted
from paper_2308_07403_b200 import workloads as wl

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 100, 257, 600])
def test_real_weights_bitwise(cuda, n):
    g = weighted(n, 0.1, 1.0, 100.0, n)
    np.testing.assert_array_equal(rb.floyd_warshall(g), orc.floyd_warshall(np.asarray(g.weights)))


def test_cfg4_shaped_weights_bitwise(cuda):
    g = wl.weighted_er_graph(700, 0.1, 1.0, 5.0, 42)
    np.testing.assert_array_equal(rb.floyd_warshall(g), orc.floyd_warshall(np.asarray(g.weights)))


def test_integer_weights_and_sparse_unreachable(cuda):
    rng = np.random.default_rng(3)
    n = 300
    present = rng.random((n, n)) < 0.004
    np.fill_diagonal(present, False)
    w = np.where(present, rng.integers(1, 9, (n, n)).astype(np.float64), np.inf)
    g = rb.Graph(n, w, rb.GraphKind.INTEGER_WEIGHTED)
    got = rb.floyd_warshall(g)
    np.testing.assert_array_equal(got, orc.floyd_warshall(w))
    assert np.isinf(got).any()
    np.testing.assert_array_equal(rb.dijkstra_apsp(g), got)


@pytest.mark.parametrize("make", [lambda: grid(9), lambda: dense(200, 0.05, 1)])
def test_unweighted_equals_bfs(cuda, make):
    g = make()
    np.testing.assert_array_equal(rb.floyd_warshall(g), rb.bfs_apsp(g))
    assert rb.graph_diameter(rb.floyd_warshall(g)) == orc.bfs_apsp(np.asarray(g.weights))[
        np.isfinite(orc.bfs_apsp(np.asarray(g.weights)))].max()
