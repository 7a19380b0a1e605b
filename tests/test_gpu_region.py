"""GPU: dense/sparse degree-threshold split (builder-defined).

No reference implementation exists; parity is pinned by
exact composition: C_sparse + exact(G[V_d]) == exact(G),
with exact(G) itself checked against the oracle.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _needle(agpm, n=1 << 14, deg=8, cliques=40, k=5, seed=3):
    return agpm.er_fast(n, n * deg // 2, seed, planted_k=k, planted_count=cliques).relabel_by_degree()


@pytest.mark.parametrize("pattern", ["triangle", "4clique", "5clique", "4cycle", "house", "5path"])
@pytest.mark.parametrize("tau", [4, 12, 40])
def test_composition_identity(agpm, oracle, pattern, tau):
    g = agpm.rmat(11, 8, seed=6).relabel_by_degree()
    dg = agpm.DeviceGraph(g)
    plan = agpm.compile_plan(pattern)
    res = agpm.region_split(dg, plan, tau, dense="exact")
    off, nbr = g.arrays()
    exact = oracle.exact_count(off, nbr, g.edge_count, plan)
    assert res.c_sparse + int(res.c_dense) == exact == agpm.exact_count(dg, plan)
    deg = np.diff(off)
    assert res.tau_id == int((deg < tau).sum())
    dense = dg.induced_suffix(res.tau_id)
    assert agpm.exact_count(dense, plan) == int(res.c_dense)


def test_oriented_clique_region(agpm):
    g = agpm.rmat(12, 16, seed=2).relabel_by_degree()
    plan = agpm.compile_plan("4clique")
    sym = agpm.region_split(agpm.DeviceGraph(g), plan, 30, dense="exact")
    ori = agpm.region_split(agpm.DeviceGraph(g.orient_by_degree()), plan, sym.tau_id, dense="exact")
    assert ori.rooted and sym.rooted
    assert (ori.c_sparse, ori.c_dense) == (sym.c_sparse, sym.c_dense)


def test_needle_found_exactly(agpm):
    """Config-4 shape: planted 5-cliques sit in the sparse region and are counted exactly."""
    g = _needle(agpm)
    dg = agpm.DeviceGraph(g)
    plan = agpm.compile_plan("5clique")
    truth = agpm.exact_count(dg, plan)
    assert truth >= 40
    for dense in ("ns", "gs", "exact"):
        res = agpm.region_split(dg, plan, 16, dense=dense, eps=0.05, max_samples=1 << 22)
        assert res.c_sparse + (res.c_dense if res.dense_exact else 0) <= truth
        if res.dense_exact or res.dense_edges == 0:
            assert res.estimate == truth


def test_rejects_unsorted_graph(agpm):
    g = agpm.rmat(10, 8, seed=6)  # not relabelled
    with pytest.raises(ValueError):
        agpm.region_split(agpm.DeviceGraph(g), agpm.compile_plan("triangle"), 8)


@pytest.mark.parametrize("core", [65536, 96, 0])
@pytest.mark.parametrize("scale,ef,tau", [(12, 16, 8), (14, 16, 30), (16, 16, 64), (16, 8, 1000)])
def test_cycle4_pair_count_equals_wedge_dfs(agpm, core, scale, ef, tau):
    """The 4-cycle C_sparse by pair aggregation (cycle4_sparse.cu: pair-core table
    + dense-core popcounts + direct wedges below the pair core) equals the rooted
    wedge DFS (exact_engine.cpp:19-62, roots < tau_id) for every pair-core size:
    the full 64 K core, a 96-id core (almost everything on the direct path) and
    no core at all (all direct, list searches only)."""
    agpm.set_core_dim(core)
    try:
        g = agpm.rmat(scale, ef, seed=scale).relabel_by_degree()
        dg = agpm.DeviceGraph(g)
        plan = agpm.compile_plan("4cycle")
        res = agpm.region_split(dg, plan, tau, dense="exact")
        assert res.rooted
        assert res.c_sparse == agpm.exact_count_rooted(dg, plan, res.tau_id)
        assert res.c_sparse + int(res.c_dense) == agpm.exact_count(dg, plan)
    finally:
        agpm.set_core_dim(None)


@pytest.mark.slow
def test_cycle4_region_split_rmat20(agpm):
    """Config-3 shape at RMAT-20: region split (tau = 64) with the exact dense leg
    composes to the full exact 4-cycle count."""
    g = agpm.rmat(20, 16, seed=1).relabel_by_degree()
    dg = agpm.DeviceGraph(g)
    plan = agpm.compile_plan("4cycle")
    res = agpm.region_split(dg, plan, 64, dense="exact")
    assert res.c_sparse + int(res.c_dense) == agpm.exact_count(dg, plan)
