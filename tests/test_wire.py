"""CPU: the edge-list and distance-CSV wire formats (graphs.py:284-329,
cli.py:204-210) against text written by the reference itself (tests/golden/wire.npz)."""

import numpy as np
import pytest

import paper_2308_07403_b200 as rb


def test_write_edge_list_matches_reference(golden, tmp_path):
    f = golden("wire")
    g = rb.Graph(12, f["weights"], rb.GraphKind.REAL_WEIGHTED)
    el = rb.edge_list_from_graph(g)
    np.testing.assert_array_equal(np.array(el.edges, dtype=np.float64), f["edges"])
    p = tmp_path / "g.txt"
    rb.write_edge_list(el, p)
    assert p.read_text() == str(f["edge_text"])


def test_read_edge_list_matches_reference(golden, tmp_path):
    f = golden("wire")
    p = tmp_path / "g.txt"
    p.write_text("# a comment\n\n" + str(f["edge_text"]) + "   # trailing\n")
    el = rb.read_edge_list(p)
    assert el.vertex_count == 12
    np.testing.assert_array_equal(np.array(el.edges, dtype=np.float64), f["edges"])
    assert rb.infer_kind(el).value == str(f["kind"])
    g = rb.graph_from_edge_list(el, rb.infer_kind(el))
    np.testing.assert_array_equal(g.weights, f["weights"])


def test_distance_csv_matches_reference(golden, tmp_path):
    f = golden("wire")
    p = tmp_path / "d.csv"
    rb.write_distance_csv(f["ring_d"], p)
    assert p.read_text() == str(f["ring_csv"])


@pytest.mark.parametrize("text", ["0 1 1.0\n", "V\n", "V 3\n0 1\n", "# only a comment\n"])
def test_read_edge_list_errors(tmp_path, text):
    p = tmp_path / "bad.txt"
    p.write_text(text)
    with pytest.raises(ValueError):
        rb.read_edge_list(p)


def test_infer_kind():
    E = rb.EdgeList
    assert rb.infer_kind(E(2, ((0, 1, 1.0),))) is rb.GraphKind.UNWEIGHTED
    assert rb.infer_kind(E(2, ((0, 1, 3.0),))) is rb.GraphKind.INTEGER_WEIGHTED
    assert rb.infer_kind(E(2, ((0, 1, 2.5),))) is rb.GraphKind.REAL_WEIGHTED
    assert rb.infer_kind(E(2, ())) is rb.GraphKind.UNWEIGHTED
