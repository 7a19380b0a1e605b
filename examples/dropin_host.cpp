// Reference-style caller compiled against the drop-in header (include/agpm/agpm.hpp)
// and linked with libagpm_b200.so. Host-only parts run anywhere; the sampling
// calls need a B200 (they throw agpm::device_error otherwise — no CPU fallback).
#include <cstdio>
#include <string>

#include "agpm/agpm.hpp"

int main(int argc, char** argv) {
  const bool device = argc > 1 && std::string(argv[1]) == "--device";
  agpm::ExecutionPlan plan = agpm::compile_plan(agpm::parse_pattern_spec("4clique"), agpm::VerifyMode::Eager);
  std::printf("plan %s k=%d steps=%zu seed_ordered=%d rule='%s'\n", plan.pattern.name.c_str(), plan.k(),
              plan.steps.size(), (int)plan.seed_ordered, plan.scaling_rule_text().c_str());
  agpm::Pattern hand;
  hand.vertex_count = 4;
  hand.edges = {{0, 1}, {1, 2}, {2, 3}, {3, 0}};
  std::printf("hand-built 4-cycle rule='%s'\n", agpm::compile_plan(hand, agpm::VerifyMode::Eager).scaling_rule_text().c_str());
  try {
    agpm::parse_pattern_spec("pentagon");
  } catch (const agpm::pattern_error& e) {
    std::printf("pattern_error ok\n");
  }
  agpm::CsrGraph g = agpm::CsrGraph::from_edges({{0, 1}, {1, 2}, {0, 2}, {2, 3}, {1, 3}, {0, 3}});
  std::printf("graph n=%u m=%llu\n", g.vertex_count(), (unsigned long long)g.edge_count());
  agpm::SampleAccumulator acc;
  acc.add(0.0, false);
  acc.add(4.0, true);
  std::printf("eps_hat=%.5f\n", agpm::predicted_error(acc, 0.05).epsilon_hat);
  // test_gs_engine.cpp:14-34: eps 0.1, delta 0.05, C 1e6, gamma 50 -> p = 0.05533, 18 colours
  agpm::KeepProbability kp = agpm::choose_keep_probability({0.1, 0.05, 1e6, 50.0});
  std::printf("keep p=%.5f colors=%u\n", kp.p, kp.color_count());
  {  // exact_engine.hpp / gs_engine.hpp / ns_engine.hpp host entry points
    agpm::Pattern tri_p = agpm::parse_pattern_spec("triangle");
    agpm::SeedIndex seeds(g.view());
    auto a0 = seeds.arc(g.view(), 0), a11 = seeds.arc(g.view(), 11);
    std::printf("brute triangles=%llu through(0,1)=%llu gamma=%llu seeds=%llu arc0=(%u,%u) arc11=(%u,%u)\n",
                (unsigned long long)agpm::brute_force_count(g, tri_p),
                (unsigned long long)agpm::count_matches_through_edge(g.view(), tri_p, 0, 1),
                (unsigned long long)agpm::estimate_gamma(g.view(), tri_p, 10, 1),
                (unsigned long long)seeds.total_arcs(), a0.first, a0.second, a11.first, a11.second);
  }
  agpm::CostCone cone = agpm::ns_cost_cone(g.view(), plan, 1000, 1e-9);
  agpm::GsCostEstimate gsm = agpm::gs_cost_estimate(g.view(), plan, 2, 1e-9, 4);
  std::printf("cone %.3e..%.3e gs %.3e -> %s\n", cone.lower_time, cone.upper_time, gsm.total_seconds,
              agpm::select_scheme(cone, gsm) == agpm::Scheme::GS ? "GS" : "NS");
  if (device) {
    agpm::OnlineResult r = agpm::run_ns_online(g.view(), plan, 0.05, 0.05, agpm::OnlinePolicy{}, 7);
    std::printf("K4 4-cliques ~ %.4f (n=%llu converged=%d)\n", r.report.mu, (unsigned long long)r.report.n,
                (int)r.report.converged);
    agpm::CounterRng rng(7, 0, 3);
    agpm::SampledCount s = agpm::draw_sample(g.view(), plan, rng);
    std::printf("draw value=%.1f hit=%d\n", s.value, (int)s.hit);
    agpm::CounterRng rng2(7, 0, 3);
    agpm::SampledCount s2 = agpm::draw_sample(g.view(), agpm::SeedIndex(g.view()), plan, rng2);
    std::printf("draw with seed index value=%.1f hit=%d\n", s2.value, (int)s2.hit);
    // freed graphs never alias new ones in the device-mirror cache (same n and m,
    // possibly the same host addresses): triangle counts must alternate 0, 1, 0, 1
    agpm::ExecutionPlan tri0 = agpm::compile_plan(agpm::parse_pattern_spec("triangle"), agpm::VerifyMode::Eager);
    std::printf("aba");
    for (int i = 0; i < 4; ++i) {
      agpm::CsrGraph a = i % 2 ? agpm::CsrGraph::from_edges({{0, 1}, {1, 2}, {0, 2}, {2, 3}})
                               : agpm::CsrGraph::from_edges({{0, 1}, {1, 2}, {2, 3}, {0, 3}});
      std::printf(" %llu", (unsigned long long)agpm::exact_count(a.view(), tri0).count);
    }
    std::printf("\n");
    agpm::OnlineResult rw = agpm::run_ns_online(g.view(), plan, 0.05, 0.05, agpm::OnlinePolicy{}, 7, 4);
    std::printf("workers=4 n=%llu same=%d\n", (unsigned long long)rw.report.n,
                (int)(rw.report.n == r.report.n && rw.accumulator.sum == r.accumulator.sum));
    // K4: 4 triangles, one 4-clique (test_exact_engine.cpp:19-25)
    agpm::ExecutionPlan tri = agpm::compile_plan(agpm::parse_pattern_spec("triangle"), agpm::VerifyMode::Eager);
    std::printf("exact triangles=%llu 4cliques=%llu\n", (unsigned long long)agpm::exact_count(g.view(), tri).count,
                (unsigned long long)agpm::exact_count(g.view(), plan).count);
    agpm::GsEstimate gs = agpm::gs_estimate(g, tri, agpm::SparsifyParams::color(1, 5));
    std::printf("gs c=1 estimate=%.1f raw=%llu\n", gs.estimate, (unsigned long long)gs.raw_count);
    agpm::ColoredCsr cc = agpm::ColoredCsr::with_colors(g, {0, 1, 0, 1}, 2);
    agpm::ColoredCsr one = cc.merge_colors({0, 0});
    std::printf("colored same=%llu merged same=%llu merged triangles=%llu\n",
                (unsigned long long)cc.same_color_edge_count(), (unsigned long long)one.same_color_edge_count(),
                (unsigned long long)one.exact_count_sparsified(tri).count);
  }
  return 0;
}
