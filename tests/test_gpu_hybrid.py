"""GPU parity for the profiler and the hybrid NS/GS choice.

fast_profile (cost_model.cpp:147-190) runs the device Bernoulli sparsifier and
the device online sampler; against the reference with threads = 1 the
converged sample count is exact and the derived estimates agree to reduction
rounding. The hybrid driver reproduces the decision the reference's own
pieces make (agpm_main.cpp:221-287).
"""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pattern,n,p,seed", [("4clique", 400, 0.3, 88001), ("triangle", 1500, 0.04, 77001),
                                               ("4cycle", 2000, 0.05, 77002), ("6clique", 400, 0.3, 88001)])
def test_fast_profile_matches_reference(agpm, ref, pattern, n, p, seed):
    g = agpm.er_graph(n, p, seed)
    rg = ref.er_graph(n, p, seed)
    plan = agpm.compile_plan(pattern)
    prof = agpm.fast_profile(agpm.DeviceGraph(g), plan, 0.3, 0.1, 99)
    out6 = (C.c_double * 6)()
    assert ref.L.ref_fast_profile(rg.h, pattern.encode(), 0.3, 0.1, 99, 1, 1000000, out6) == 0
    assert prof.reliable == int(out6[5]) and prof.n_converged == int(out6[4])
    for mine, theirs in [(prof.n_samples_estimate, out6[0]), (prof.mu_prime, out6[1]), (prof.scaled_count, out6[2]),
                         (prof.epsilon_hat_final, out6[3])]:
        assert mine == theirs or abs(mine - theirs) <= 1e-9 * max(1.0, abs(theirs))


@pytest.mark.parametrize("pattern,n,p,seed", [("4clique", 400, 0.3, 88001), ("6clique", 400, 0.3, 88001),
                                               ("4cycle", 1500, 0.04, 77001)])
def test_hybrid_decision_matches_reference_pieces(agpm, ref, pattern, n, p, seed):
    g = agpm.er_graph(n, p, seed)
    rg = ref.er_graph(n, p, seed)
    plan = agpm.compile_plan(pattern)
    hw = 1e-9
    res = agpm.count_hybrid(g, agpm.DeviceGraph(g), plan, 0.1, 0.99, seed=7, profile_fraction=0.3, hw_const=hw)
    # the reference's pieces, threads = 1 (agpm_main.cpp:221-287)
    out6 = (C.c_double * 6)()
    ref.L.ref_fast_profile(rg.h, pattern.encode(), 0.3, 0.1, 7, 1, 1000000, out6)
    if not out6[5]:
        assert res.decision == 0
        return
    gam = C.c_uint64()
    ref.L.ref_estimate_gamma(rg.h, pattern.encode(), min(1000, max(rg.info()[1], 1)), 7 + 17, 50000000, C.byref(gam))
    gamma = 2.0 * max(1, gam.value)
    kp, useless, colors = C.c_double(), C.c_int(), C.c_uint32()
    ref.L.ref_choose_keep_probability(0.1, 0.01, out6[2], gamma, C.byref(kp), C.byref(useless), C.byref(colors))
    cone5 = (C.c_double * 5)()
    ref.L.ref_ns_cost_cone(rg.h, pattern.encode(), max(1, int(out6[0])), hw, cone5)
    gs3 = (C.c_double * 3)()
    ref.L.ref_gs_cost_estimate(rg.h, pattern.encode(), max(2, colors.value), hw, ref.triangle_count(rg), gs3)
    want = 1 if gs3[2] < cone5[3] else 0
    assert res.gamma == gamma and res.keep.color_count == colors.value
    assert res.decision == want
    truth = agpm.exact_count(agpm.DeviceGraph(g), plan)
    if res.decision == 0:
        assert res.ns.report.converged
    assert truth > 0 and abs(res.estimate - truth) / truth < 0.5
