"""Host-side logic of the drop-in API that needs no GPU (argument contract,
Graph accessors, scalar helpers) -- semantics of the reference's
test_expected_force.py:29-66,108-135 and test_graph.py:96-118."""
import math

import numpy as np
import pytest

import paper_2306_00606_b200 as efg
from paper_2306_00606_b200.graph import Graph


def graph_of(case):
    return Graph(case.n, case.m, case.get("offsets"), case.get("neighbors"), case.get("orig_ids"))


def test_argument_errors_raise_value_error(golden):
    g = graph_of(golden["path3"])
    with pytest.raises(ValueError):
        efg.ef_cluster_centric(g, workers=0)
    with pytest.raises(ValueError):
        efg.ef_cluster_centric(g, chunk_size=0)
    with pytest.raises(ValueError):
        efg.ef_vertex_centric(g, workers=0)
    with pytest.raises(ValueError):
        efg.ef(g, mode="edge_centric")


def test_empty_graph_needs_no_device():
    g = Graph(0, 0, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.int64))
    r = efg.ef_cluster_centric(g)
    assert r.ef.size == 0 and r.cluster_total.dtype == np.int64 and r.flags.dtype == np.uint8
    assert r.clusters_processed == 0
    assert efg.build_graph([]).n == 0
    assert efg.build_graph(np.zeros((0, 2), np.int64)).n == 0


def test_cluster_degree(golden):
    tri = graph_of(golden["triangle"])
    assert efg.cluster_degree(tri, 0, 1, 2) == 0
    assert efg.cluster_degree(graph_of(golden["path3"]), 0, 1, 2) == 0
    assert efg.cluster_degree(graph_of(golden["star3"]), 1, 0, 2) == 1
    p4 = graph_of(golden["path4"])
    with pytest.raises(ValueError):
        efg.cluster_degree(p4, 0, 1, 1)
    with pytest.raises(ValueError):
        efg.cluster_degree(p4, 0, 1, 3)


def test_entropy_from_histogram():
    assert efg.entropy_from_histogram({1: 6}) == pytest.approx(math.log(6), abs=1e-12)
    assert efg.entropy_from_histogram({}) == 0.0
    assert efg.entropy_from_histogram({0: 4}) == 0.0
    assert efg.entropy_from_histogram({1: 2, 2: 1}) == pytest.approx(1.5 * math.log(2), abs=1e-12)
    assert efg.entropy_from_histogram({0: 10, 1: 6}) == pytest.approx(math.log(6), abs=1e-12)
    with pytest.raises(ValueError):
        efg.entropy_from_histogram({-1: 2})


def test_graph_accessors(golden):
    tri = graph_of(golden["triangle"])
    assert tri.degree(0) == 2 and tri.has_edge(0, 2)
    p3 = graph_of(golden["path3"])
    assert not p3.has_edge(0, 2) and not p3.has_edge(1, 1)
    assert graph_of(golden["star3"]).avg_degree() == 6 / 4
    with pytest.raises(ValueError):
        p3.degree(3)
    with pytest.raises(ValueError):
        p3.adjacency(-1)
    with pytest.raises(ValueError):
        p3.has_edge(0, 99)
    rel = graph_of(golden["relabel"])
    assert rel.relabeling == {5: 0, 9: 1}
    assert efg.cluster_count(graph_of(golden["star3"])) == 3


def test_rmat_params_validation():
    with pytest.raises(ValueError):
        efg.RmatParams(scale=0, avg_degree=1)
    with pytest.raises(ValueError):
        efg.RmatParams(scale=4, avg_degree=0)
    with pytest.raises(ValueError):
        efg.RmatParams(scale=4, avg_degree=2, quadrant_probs=(0.5, 0.5, 0.5, 0.5))


def test_key_nodes_argument_contract():
    with pytest.raises(ValueError):
        efg.key_nodes(np.zeros(4), k=1, frac=0.5)
    with pytest.raises(ValueError):
        efg.key_nodes(np.zeros(4))
    assert efg.key_nodes(np.zeros(4), k=0).size == 0


def test_write_ef_csv_format(golden):
    import io
    case = golden["star3"]
    g = graph_of(case)
    r = efg.EFResult(case.get("ef"), case.get("cluster_total"), case.get("flags"), 3)
    buf = io.StringIO()
    efg.write_ef_csv(g, r, buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == "node,ef,cluster_total"
    assert lines[1] == f"0,{math.log(6):.9g},6"
