"""GPU: device graph ingest (graph_build.cu) is bit-identical to the host builders.

Host twins: CsrGraph::from_edges (csr_graph.cpp:46-72), the RMAT / ER generators,
relabel_by_degree and orient_by_degree (csr_graph.cpp:172). Every device-built
view is downloaded and compared array for array with the host-built one, then
sampled: identical seed arcs and `up` counts give identical accumulators.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(dg, hg, oriented=False):
    off, nbr = hg.arrays()
    b, e, nb = dg.download()
    info = dg.info()
    assert info["vertex_count"] == hg.vertex_count
    assert info["edge_count"] == hg.edge_count
    assert info["arcs"] == len(nbr)
    assert info["oriented"] == oriented
    np.testing.assert_array_equal(b, off[:-1])
    np.testing.assert_array_equal(e, off[1:])
    np.testing.assert_array_equal(nb, nbr)


def _same_samples(agpm, dg, hg, pattern="4clique", budget=1 << 15):
    plan = agpm.compile_plan(pattern)
    a = agpm.run_fixed_budget(dg, plan, budget, 7)
    b = agpm.run_fixed_budget(agpm.DeviceGraph(hg), plan, budget, 7)
    assert (a.n, a.hits, a.sum, a.squared_sum) == (b.n, b.hits, b.sum, b.squared_sum)


@pytest.mark.parametrize("scale,ef,relabel", [(10, 8, False), (12, 16, True), (16, 16, False), (16, 16, True)])
def test_rmat_device(agpm, scale, ef, relabel):
    dg = agpm.rmat_device(scale, ef, seed=3, relabel=relabel)
    hg = agpm.rmat(scale, ef, seed=3)
    if relabel:
        hg = hg.relabel_by_degree()
    _same(dg, hg)
    assert dg.info()["max_degree"] == hg.max_degree()
    _same_samples(agpm, dg, hg)


@pytest.mark.parametrize("relabel", [False, True])
def test_er_fast_device_planted(agpm, relabel):
    n = 1 << 14
    dg = agpm.er_fast_device(n, n * 4, seed=4, planted_k=5, planted_count=50, relabel=relabel)
    hg = agpm.er_fast(n, n * 4, seed=4, planted_k=5, planted_count=50)
    if relabel:
        hg = hg.relabel_by_degree()
    _same(dg, hg)
    _same_samples(agpm, dg, hg, "5clique")


def test_from_edges_device_loops_duplicates(agpm):
    rng = np.random.default_rng(11)
    pairs = rng.integers(0, 300, size=(5000, 2), dtype=np.uint32)
    pairs[::17, 1] = pairs[::17, 0]  # self-loops
    pairs = np.concatenate([pairs, pairs[:1000, ::-1]])  # reversed duplicates
    for relabel in (False, True):
        dg = agpm.graph_from_edges_device(pairs, min_vertex_count=0, relabel=relabel)
        hg = agpm.CsrGraph.from_edges(pairs)
        if relabel:
            hg = hg.relabel_by_degree()
        _same(dg, hg)


@pytest.mark.parametrize("pairs,minv", [
    (np.zeros((0, 2), np.uint32), 0),
    (np.zeros((0, 2), np.uint32), 5),
    (np.array([[3, 3], [4, 4]], np.uint32), 0),  # loops only: n from the ids, no edges
    (np.array([[0, 1]], np.uint32), 10),          # isolated tail vertices
    (np.array([[9, 8], [8, 9], [9, 8]], np.uint32), 0),
])
def test_from_edges_device_edge_cases(agpm, pairs, minv):
    dg = agpm.graph_from_edges_device(pairs, min_vertex_count=minv)
    hg = agpm.CsrGraph.from_edges(pairs, minv)
    _same(dg, hg)
    dr = agpm.graph_from_edges_device(pairs, min_vertex_count=minv, relabel=True)
    _same(dr, hg.relabel_by_degree())


def test_relabel_and_orient_device(agpm):
    hg = agpm.rmat(14, 16, seed=5)
    dg = agpm.DeviceGraph(hg)
    _same(dg.relabel_by_degree(), hg.relabel_by_degree())
    _same(dg.orient_by_degree(), hg.orient_by_degree(), oriented=True)
    rl = hg.relabel_by_degree()
    od = agpm.DeviceGraph(rl).orient_by_degree()
    _same(od, rl.orient_by_degree(), oriented=True)
    # exact count on the device-oriented DAG == on the host-oriented one
    plan = agpm.compile_plan("4clique")
    assert agpm.exact_count(od, plan) == agpm.exact_count(agpm.DeviceGraph(rl.orient_by_degree()), plan)
    with pytest.raises(Exception):
        od.orient_by_degree()  # already oriented


@pytest.mark.slow
def test_rmat22_device_matches_host(agpm):
    """config 3's graph (RMAT-22 ef16, relabelled): device build == host build."""
    dg = agpm.rmat_device(22, 16, seed=1, relabel=True)
    hg = agpm.rmat(22, 16, seed=1).relabel_by_degree()
    _same(dg, hg)
