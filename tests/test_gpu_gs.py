"""GPU parity for sparsification and GS.

Colour split: colours, split ends, the stably partitioned neighbour array and the
same-colour edge count equal ColoredCsr::color_vertices (colored_csr.cpp:14-54);
Bernoulli: the kept CSR equals bernoulli_sparsify (csr_graph.cpp:190-213);
gs_estimate: raw counts bit-exact, scale/estimate equal (gs_engine.cpp:42-75).
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_color_split_matches_reference_golden(agpm):
    import hashlib
    with open(os.path.join(GOLDEN, "counts.json")) as f:
        g = json.load(f)["split"]
    dg = agpm.DeviceGraph(agpm.er_graph(60, 0.2, 17))
    for key, r in g.items():
        c, seed = map(int, key.split("|"))
        view, colors, same = dg.color_split(c, seed)
        b, e, nb = view.download()
        assert colors.tolist() == r["colors"] and e.tolist() == r["split_end"] and same == r["same_edges"]
        assert hashlib.sha256(np.ascontiguousarray(nb).tobytes()).hexdigest()[:32] == r["nbr_hash"]


@pytest.mark.parametrize("c,seed", [(1, 3), (2, 5), (4, 19), (7, 123)])
def test_color_split_matches_oracle(agpm, oracle, c, seed):
    g = agpm.rmat(12, 16, seed=2).relabel_by_degree()
    off, nbr = g.arrays()
    colors, split, out, same = oracle.color_split(off, nbr, c, seed)
    view, dcolors, dsame = agpm.DeviceGraph(g).color_split(c, seed)
    b, e, nb = view.download()
    assert np.array_equal(dcolors, colors) and np.array_equal(e, split) and np.array_equal(nb, out)
    assert dsame == same == view.info()["edge_count"]


@pytest.mark.parametrize("p,seed", [(1.0, 5), (0.5, 7), (0.1, 11), (0.9, 3)])
def test_bernoulli_matches_oracle(agpm, oracle, p, seed):
    g = agpm.rmat(12, 16, seed=2)
    off, nbr = g.arrays()
    ooff, onbr = oracle.bernoulli_sparsify(off, nbr, p, seed)
    sp = agpm.DeviceGraph(g).bernoulli_sparsify(p, seed)
    b, e, nb = sp.download()
    assert np.array_equal(b, ooff[:-1]) and np.array_equal(e, ooff[1:]) and np.array_equal(nb[: len(onbr)], onbr)
    assert sp.info()["edge_count"] == len(onbr) // 2
    with pytest.raises(ValueError):
        agpm.DeviceGraph(g).bernoulli_sparsify(0.0, 1)


def test_gs_estimate_matches_reference_golden(agpm):
    with open(os.path.join(GOLDEN, "counts.json")) as f:
        gold = json.load(f)
    dg = agpm.DeviceGraph(agpm.er_graph(200, 0.08, 71))
    for pat, per_c in gold["colored"].items():
        for c, cnt in per_c.items():
            r = agpm.gs_estimate(dg, agpm.compile_plan(pat), "color", colors=int(c), seed=7)
            assert r.raw_count == cnt, (pat, c)
    for pat, r in gold["gs"].items():
        plan = agpm.compile_plan(pat)
        c4 = agpm.gs_estimate(dg, plan, "color", colors=4, seed=11)
        b5 = agpm.gs_estimate(dg, plan, "bernoulli", keep_probability=0.5, seed=11)
        assert [c4.estimate, c4.raw_count, c4.scale] == r["color4"]
        assert [b5.estimate, b5.raw_count, b5.scale] == r["bern05"]


def test_gs_errors_and_identities(agpm):
    g = agpm.er_graph(60, 0.2, 17)
    dg = agpm.DeviceGraph(g)
    with pytest.raises(ValueError):  # gs_engine.cpp:44-47
        agpm.gs_estimate(dg, agpm.compile_plan("4motif-path"), "bernoulli", keep_probability=0.5, seed=1)
    for pat in ["triangle", "4cycle", "house"]:  # c = 1 / p = 1 reproduce exact (test_gs_engine.cpp:36-47)
        plan = agpm.compile_plan(pat)
        exact = agpm.exact_count(dg, plan)
        assert agpm.gs_estimate(dg, plan, "color", colors=1, seed=5).estimate == exact
        assert agpm.gs_estimate(dg, plan, "bernoulli", keep_probability=1.0, seed=5).estimate == exact


def test_triangle_count(agpm, oracle):
    with open(os.path.join(GOLDEN, "counts.json")) as f:
        tri = json.load(f)["triangle_count"]
    for key, cnt in tri.items():
        _, n, p, s = key.split("|")
        g = agpm.er_graph(int(n), float(p), int(s))
        assert agpm.DeviceGraph(g).triangle_count() == cnt
        assert agpm.DeviceGraph(g.orient_by_degree()).triangle_count() == cnt


@pytest.mark.parametrize("c,seed,group_map", [(4, 19, [0, 1, 2, 3]), (4, 19, [0, 0, 0, 0]), (4, 19, [0, 0, 1, 1]),
                                             (6, 7, [2, 0, 1, 1, 0, 2]), (5, 3, [0, 1, 0, 1, 0])])
def test_merge_colors_matches_reference(agpm, ref, c, seed, group_map):
    """ColoredCsr::merge_colors (colored_csr.cpp:56-88) against the compiled
    reference: coarse colours, split ends, the permuted neighbour array and the
    same-colour edge count are identical (identity / merge-to-one / pairwise
    cases of test_graph_core.cpp:267-298 plus uneven maps)."""
    g = agpm.rmat(11, 16, seed=2).relabel_by_degree()
    off, nbr = g.arrays()
    rg = ref.from_csr(off, nbr, g.edge_count)
    rcol, rsplit, rnbr, rsame = ref.merge_colors(rg, c, seed, group_map)
    dg = agpm.DeviceGraph(g)
    _, fine, _ = dg.color_split(c, seed)
    view, coarse, same = dg.merge_colors(fine, c, group_map)
    b, e, nb = view.download()
    assert np.array_equal(coarse, rcol) and np.array_equal(e, rsplit) and np.array_equal(nb, rnbr)
    assert same == rsame == view.info()["edge_count"]


def test_merge_colors_errors(agpm):
    g = agpm.er_graph(40, 0.2, 3)
    dg = agpm.DeviceGraph(g)
    _, fine, _ = dg.color_split(4, 1)
    with pytest.raises(ValueError):
        dg.merge_colors(fine, 4, [0, 2, 2, 2])  # gap at 1 (test_graph_core.cpp:297)
    with pytest.raises(ValueError):
        dg.merge_colors(fine, 4, [0, 1])  # not total (:298)
    with pytest.raises(ValueError):
        dg.color_split_with_colors(np.full(40, 9, np.uint32), 4)  # colour out of range


@pytest.mark.parametrize("pattern,colors", [("triangle", 2), ("4clique", 2), ("4cycle", 3)])
def test_gs_online_replay_and_bound(agpm, oracle, pattern, colors):
    """Colour GS run to a relative error bound (Appendix C.2): the stop index,
    the accumulated estimates and the report equal a host replay of the same
    colourings (gs_estimate with seeds derive_key(seed, i, 0)) through the
    reference's window rule, and the estimate sits within 3 eps of the exact count."""
    g = agpm.er_graph(400, 0.05, 8).relabel_by_degree()
    dg = agpm.DeviceGraph(g)
    plan = agpm.compile_plan(pattern)
    exact = agpm.exact_count(dg, plan)
    eps, delta, seed = 0.05, 0.05, 3
    r = agpm.gs_online(dg, plan, colors, eps, delta, max_colorings=4000, seed=seed)
    assert r.report.converged and 2 <= r.windows < 4000
    s = sq = 0.0
    for i in range(r.windows):
        x = agpm.gs_estimate(dg, plan, "color", colors=colors, seed=oracle.L.orc_derive_key(seed, i, 0)).estimate
        s += x
        sq += x * x
        rep = oracle.predicted_error(agpm.Accumulator(i + 1, 0, s, sq), delta)
        assert (rep.epsilon_hat <= eps) == (i + 1 == r.windows)
    assert s == r.accumulator.sum and sq == r.accumulator.squared_sum and r.report.mu == s / r.windows
    assert abs(r.report.mu - exact) <= 3 * eps * exact
    with pytest.raises(ValueError):
        agpm.gs_online(dg, plan, colors, 1.5, delta)
