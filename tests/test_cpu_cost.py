"""CPU: hybrid-selection host logic against the compiled reference.

Keep probability (gs_engine.cpp:24-40), NS cost cone (cost_model.cpp:78-110),
GS cost model (:112-145), gamma probing (gs_engine.cpp:179-197,
exact_engine.cpp:135-213): same inputs, same outputs (doubles bit-equal).
"""
import ctypes as C

import pytest

PATTERNS = ["triangle", "4clique", "4cycle", "house", "5path", "4motif-path", "dumbbell"]


def test_keep_probability(agpm, ref):
    for args in [(0.1, 0.05, 1e6, 50.0), (0.1, 0.05, 10.0, 50.0), (0.1, 0.05, 1e7, 20.0), (0.1, 0.05, 0.0, 50.0),
                 (0.01, 0.01, 3.3e9, 7.0), (0.5, 0.2, 12345.0, 3.0)]:
        k = agpm.choose_keep_probability(*args)
        p, useless, colors = C.c_double(), C.c_int(), C.c_uint32()
        assert ref.L.ref_choose_keep_probability(*args, C.byref(p), C.byref(useless), C.byref(colors)) == 0
        assert (k.p, k.sparsification_useless, k.color_count) == (p.value, useless.value, colors.value)
    k = agpm.choose_keep_probability(0.1, 0.05, 1e6, 50.0)
    assert abs(k.p - 0.05533) < 2e-3 * 0.05533 and k.color_count == 18  # test_gs_engine.cpp:14-34
    with pytest.raises(ValueError):
        agpm.choose_keep_probability(0.1, 0.05, 1e6, 0.0)


@pytest.mark.parametrize("pattern", PATTERNS)
def test_cost_models(agpm, ref, pattern):
    g = agpm.er_graph(300, 0.05, 55)
    rg = ref.er_graph(300, 0.05, 55)
    plan = agpm.compile_plan(pattern)
    hw = 2.5e-9
    cone = agpm.ns_cost_cone(g.vertex_count, g.arc_count, plan, 12345, hw)
    out5 = (C.c_double * 5)()
    assert ref.L.ref_ns_cost_cone(rg.h, pattern.encode(), 12345, hw, out5) == 0
    assert [cone.lower_slope, cone.upper_slope, cone.n_samples, cone.lower_time, cone.upper_time] == list(out5)
    tri = ref.triangle_count(rg)
    for colors in (1, 2, 7):
        gs = agpm.gs_cost_estimate(g.vertex_count, g.edge_count, plan, colors, hw, tri)
        out3 = (C.c_double * 3)()
        assert ref.L.ref_gs_cost_estimate(rg.h, pattern.encode(), colors, hw, tri, out3) == 0
        assert [gs.preprocess_work, gs.search_work, gs.total_seconds] == list(out3)
        assert agpm.select_scheme(cone, gs) == ("gs" if out3[2] < out5[3] else "ns")


@pytest.mark.parametrize("pattern", ["triangle", "4clique", "5path", "4cycle", "house"])
def test_gamma_probing(agpm, ref, pattern):
    g = agpm.er_graph(100, 0.1, 31)
    rg = ref.er_graph(100, 0.1, 31)
    plan = agpm.compile_plan(pattern)
    out = C.c_uint64()
    for u, v in [(0, 1), (3, 7), (10, 44), (5, 6)]:
        assert ref.L.ref_count_through_edge(rg.h, pattern.encode(), u, v, C.byref(out)) == 0
        assert agpm.count_matches_through_edge(g, plan, u, v) == out.value
    for probes, seed, budget in [(200, 5, 50000000), (50, 9, 20000)]:
        assert ref.L.ref_estimate_gamma(rg.h, pattern.encode(), probes, seed, budget, C.byref(out)) == 0
        assert agpm.estimate_gamma(g, plan, probes, seed, budget) == out.value
    k5 = agpm.CsrGraph.from_edges([(i, j) for i in range(5) for j in range(i + 1, 5)])
    assert agpm.count_matches_through_edge(k5, agpm.compile_plan("triangle"), 0, 1) == 3  # test_exact_engine.cpp:105
