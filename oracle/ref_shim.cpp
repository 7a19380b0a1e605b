// TEST INFRASTRUCTURE ONLY — never part of the product path.
//
// extern "C" shim over the UNMODIFIED reference library (agpm), compiled from
// the reference's own sources under /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libagpm_ref.so. Only tests/, smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it: it is the
// checker and the CPU baseline, never the thing measured as the product.
//
// Every function forwards to the reference's public API; the one place the
// shim re-walks reference logic (ref_draw_records) captures per-sample
// bindings through the reference's own walker (walker.hpp:30-83) and asserts
// the value/hit it reproduces equals agpm::draw_sample's.

#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "agpm/colored_csr.hpp"
#include "agpm/cost_model.hpp"
#include "agpm/csr_graph.hpp"
#include "agpm/exact_engine.hpp"
#include "agpm/gs_engine.hpp"
#include "agpm/ns_engine.hpp"
#include "agpm/pattern.hpp"
#include "agpm/plan.hpp"
#include "agpm/rng.hpp"
#include "agpm/stats.hpp"
#include "agpm/walker.hpp"
#include "agpm_b200.h"
#include "support/test_graphs.hpp"

using namespace agpm;

namespace {

std::string g_err;  // single-threaded test harness

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const pattern_error& e) {
    g_err = e.what();
    return AGPM_E_PATTERN;
  } catch (const io_error& e) {
    g_err = e.what();
    return AGPM_E_IO;
  } catch (const parse_error& e) {
    g_err = e.what();
    return AGPM_E_PARSE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return AGPM_E_INVALID;
  } catch (const std::exception& e) {
    g_err = e.what();
    return AGPM_E_INTERNAL;
  }
}

struct RefGraph {
  CsrGraph g;
};

ExecutionPlan plan_of(const char* spec, const char* induced, int mode, int sym) {
  Pattern p = parse_pattern_spec(spec, induced ? induced : "");
  return compile_plan(p, mode ? VerifyMode::Lazy : VerifyMode::Eager, sym != 0);
}

void export_plan(const ExecutionPlan& plan, agpm_plan* out) {
  std::memset(out, 0, sizeof(*out));
  std::snprintf(out->name, sizeof(out->name), "%s", plan.pattern.name.c_str());
  out->k = plan.pattern.vertex_count;
  out->induced = plan.pattern.induced == InducedMode::Vertex;
  out->n_edges = static_cast<int32_t>(plan.pattern.edges.size());
  for (size_t i = 0; i < plan.pattern.edges.size(); ++i) {
    out->edges[i][0] = plan.pattern.edges[i].first;
    out->edges[i][1] = plan.pattern.edges[i].second;
  }
  for (int v = 0; v < plan.pattern.vertex_count; ++v) out->adjacency[v] = plan.pattern.adjacency[v];
  out->verify_mode = plan.verify_mode == VerifyMode::Lazy;
  for (size_t i = 0; i < plan.order.size(); ++i) out->order[i] = plan.order[i];
  for (size_t i = 0; i < plan.pos_of.size(); ++i) out->pos_of[i] = plan.pos_of[i];
  out->seed_ordered = plan.seed_ordered;
  out->symmetry_enabled = plan.symmetry_enabled;
  out->n_steps = static_cast<int32_t>(plan.steps.size());
  for (size_t s = 0; s < plan.steps.size(); ++s) {
    const PlanStep& st = plan.steps[s];
    agpm_plan_step& o = out->steps[s];
    o.pattern_vertex = st.pattern_vertex;
    o.n_in = static_cast<int32_t>(st.in_positions.size());
    for (size_t i = 0; i < st.in_positions.size(); ++i) o.in_positions[i] = st.in_positions[i];
    o.n_out = static_cast<int32_t>(st.out_positions.size());
    for (size_t i = 0; i < st.out_positions.size(); ++i) o.out_positions[i] = st.out_positions[i];
    o.n_gt = static_cast<int32_t>(st.greater_than.size());
    for (size_t i = 0; i < st.greater_than.size(); ++i) o.greater_than[i] = st.greater_than[i];
    o.n_lt = static_cast<int32_t>(st.less_than.size());
    for (size_t i = 0; i < st.less_than.size(); ++i) o.less_than[i] = st.less_than[i];
    o.tree_parent = st.tree_parent;
    o.n_verify = static_cast<int32_t>(st.verify_edges.size());
    for (size_t i = 0; i < st.verify_edges.size(); ++i) {
      o.verify_edges[i][0] = st.verify_edges[i].first;
      o.verify_edges[i][1] = st.verify_edges[i].second;
    }
  }
  auto pairs = [](const std::vector<std::pair<int, int>>& v, int32_t* n, int32_t (*dst)[2]) {
    *n = static_cast<int32_t>(v.size());
    for (size_t i = 0; i < v.size(); ++i) {
      dst[i][0] = v[i].first;
      dst[i][1] = v[i].second;
    }
  };
  pairs(plan.closure_edges, &out->n_closure, out->closure_edges);
  pairs(plan.constraints, &out->n_constraints, out->constraints);
  pairs(plan.terminal_constraints, &out->n_terminal, out->terminal_constraints);
}

void put_acc(const SampleAccumulator& a, agpm_accumulator* o) {
  o->n = a.n;
  o->hits = a.hits;
  o->sum = a.sum;
  o->squared_sum = a.squared_sum;
}

void put_rep(const ConvergenceReport& r, agpm_report* o) {
  o->mu = r.mu;
  o->sigma = r.sigma;
  o->epsilon_hat = r.epsilon_hat;
  o->n = r.n;
  o->converged = r.converged;
  o->hit_rate = r.hit_rate;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- rng
void ref_rng_u64(uint64_t seed, uint64_t s1, uint64_t s2, uint64_t count, uint64_t* out) {
  CounterRng rng(seed, s1, s2);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng.next_u64();
}
void ref_rng_below(uint64_t seed, uint64_t s1, uint64_t s2, uint64_t bound, uint64_t count,
                   uint64_t* out) {
  CounterRng rng(seed, s1, s2);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng.next_below(bound);
}
void ref_rng_double(uint64_t seed, uint64_t s1, uint64_t s2, uint64_t count, double* out) {
  CounterRng rng(seed, s1, s2);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng.next_double();
}
uint64_t ref_derive_key(uint64_t seed, uint64_t s1, uint64_t s2) { return derive_key(seed, s1, s2); }
int ref_edge_keep(uint64_t seed, uint32_t u, uint32_t v, double p) {
  return edge_keep_decision(seed, u, v, p);
}
uint32_t ref_vertex_color(uint64_t seed, uint32_t v, uint32_t c) {
  return vertex_color_decision(seed, v, c);
}

// ---------------------------------------------------------------- stats
double ref_norm_cdf(double z) { return norm_cdf(z); }
int ref_inv_norm_cdf(double q, double* out) {
  return guard([&] { *out = inv_norm_cdf(q); });
}
int ref_predicted_error(const agpm_accumulator* acc, double delta, agpm_report* out) {
  return guard([&] {
    SampleAccumulator a;
    a.n = acc->n;
    a.hits = acc->hits;
    a.sum = acc->sum;
    a.squared_sum = acc->squared_sum;
    put_rep(predicted_error(a, delta), out);
  });
}

// ---------------------------------------------------------------- patterns / plans
int ref_plan_compile(const char* spec, const char* induced, int mode, int sym, agpm_plan* out) {
  return guard([&] { export_plan(plan_of(spec, induced, mode, sym), out); });
}
int ref_plan_scaling_rule(const char* spec, const char* induced, int mode, int sym, char* buf,
                          size_t cap) {
  return guard([&] {
    std::snprintf(buf, cap, "%s", plan_of(spec, induced, mode, sym).scaling_rule_text().c_str());
  });
}
int ref_automorphism_count(const char* spec, const char* induced, uint64_t* out) {
  return guard([&] { *out = parse_pattern_spec(spec, induced ? induced : "").automorphisms().size(); });
}
int ref_builtin_names(char* buf, size_t cap) {
  std::string s;
  for (const auto& n : builtin_pattern_names()) s += n + "\n";
  std::snprintf(buf, cap, "%s", s.c_str());
  return 0;
}

// ---------------------------------------------------------------- graphs
void ref_graph_free(RefGraph* g) { delete g; }
int ref_graph_from_edges(const uint32_t* edges, uint64_t n_edges, uint32_t min_n, RefGraph** out) {
  return guard([&] {
    std::vector<std::pair<uint32_t, uint32_t>> e(n_edges);
    for (uint64_t i = 0; i < n_edges; ++i) e[i] = {edges[2 * i], edges[2 * i + 1]};
    *out = new RefGraph{CsrGraph::from_edges(std::move(e), min_n)};
  });
}
int ref_graph_from_csr(uint32_t n, uint64_t m, const uint64_t* offsets, const uint32_t* nbr,
                       int oriented, RefGraph** out) {
  return guard([&] {
    std::vector<uint64_t> off(offsets, offsets + n + 1);
    std::vector<uint32_t> nb(nbr, nbr + off.back());
    *out = new RefGraph{CsrGraph(n, std::move(off), std::move(nb), m, oriented != 0)};
  });
}
int ref_graph_er(uint32_t n, double p, uint64_t seed, RefGraph** out) {
  return guard([&] { *out = new RefGraph{agpm::testing::er_graph(n, p, seed)}; });
}
int ref_graph_complete(uint32_t n, RefGraph** out) {
  return guard([&] { *out = new RefGraph{agpm::testing::complete_graph(n)}; });
}
int ref_graph_cycle(uint32_t n, RefGraph** out) {
  return guard([&] { *out = new RefGraph{agpm::testing::cycle_graph(n)}; });
}
int ref_graph_path(uint32_t n, RefGraph** out) {
  return guard([&] { *out = new RefGraph{agpm::testing::path_graph(n)}; });
}
int ref_graph_star(uint32_t leaves, RefGraph** out) {
  return guard([&] { *out = new RefGraph{agpm::testing::star_graph(leaves)}; });
}
int ref_graph_load(const char* path, RefGraph** out) {
  return guard([&] { *out = new RefGraph{load_graph_auto(path)}; });
}
int ref_graph_write_binary(const RefGraph* g, const char* path) {
  return guard([&] { write_binary_csr(g->g, path); });
}
int ref_graph_orient(const RefGraph* g, RefGraph** out) {
  return guard([&] { *out = new RefGraph{orient_by_degree(g->g)}; });
}
int ref_graph_bernoulli(const RefGraph* g, double p, uint64_t seed, RefGraph** out) {
  return guard([&] { *out = new RefGraph{bernoulli_sparsify(g->g, p, seed)}; });
}
void ref_graph_info(const RefGraph* g, uint32_t* n, uint64_t* m, uint64_t* arcs, int* oriented) {
  *n = g->g.vertex_count();
  *m = g->g.edge_count();
  *arcs = g->g.offsets().back();
  *oriented = g->g.oriented();
}
void ref_graph_arrays(const RefGraph* g, uint64_t* offsets, uint32_t* nbr) {
  std::memcpy(offsets, g->g.offsets().data(), g->g.offsets().size() * sizeof(uint64_t));
  std::memcpy(nbr, g->g.neighbors().data(), g->g.neighbors().size() * sizeof(uint32_t));
}
uint64_t ref_triangle_count(const RefGraph* g) { return triangle_count(g->g); }

// ColoredCsr::color_vertices (colored_csr.cpp:48-54): colors[n], split_end[n],
// permuted neighbours[arcs], same-colour edge count.
int ref_color_split(const RefGraph* g, uint32_t c, uint64_t seed, uint32_t* colors,
                    uint64_t* split_end, uint32_t* nbr, uint64_t* same_edges) {
  return guard([&] {
    ColoredCsr cc = ColoredCsr::color_vertices(g->g, c, seed);
    std::memcpy(colors, cc.colors().data(), cc.colors().size() * sizeof(uint32_t));
    std::memcpy(split_end, cc.split_end().data(), cc.split_end().size() * sizeof(uint64_t));
    std::memcpy(nbr, cc.base().neighbors().data(), cc.base().neighbors().size() * sizeof(uint32_t));
    *same_edges = cc.same_color_edge_count();
  });
}

// ColoredCsr::color_vertices(c, seed).merge_colors(group_map) (colored_csr.cpp:56-88):
// coarse colours[n], split_end[n], permuted neighbours[arcs], same-colour edges.
int ref_merge_colors(const RefGraph* g, uint32_t c, uint64_t seed, const uint32_t* group_map, uint32_t map_len,
                     uint32_t* colors, uint64_t* split_end, uint32_t* nbr, uint64_t* same_edges) {
  return guard([&] {
    ColoredCsr cc = ColoredCsr::color_vertices(g->g, c, seed)
                        .merge_colors(std::vector<uint32_t>(group_map, group_map + map_len));
    std::memcpy(colors, cc.colors().data(), cc.colors().size() * sizeof(uint32_t));
    std::memcpy(split_end, cc.split_end().data(), cc.split_end().size() * sizeof(uint64_t));
    std::memcpy(nbr, cc.base().neighbors().data(), cc.base().neighbors().size() * sizeof(uint32_t));
    *same_edges = cc.same_color_edge_count();
  });
}

// ---------------------------------------------------------------- NS engine
// Per-sample records for ids [first, first+count) of stream (seed, worker, id):
// value, hit, bindings (k per sample, 0xffffffff past a miss). Bindings come
// from re-walking draw_one (ns_engine.cpp:27-53) with the reference walker;
// the value/hit are cross-checked against agpm::draw_sample.
int ref_draw_records(const RefGraph* g, const char* spec, const char* induced, int mode, int sym,
                     uint64_t seed, uint64_t worker, uint64_t first, uint64_t count,
                     double* values, uint8_t* hits, uint32_t* bindings) {
  return guard([&] {
    ExecutionPlan plan = plan_of(spec, induced, mode, sym);
    CsrView view = g->g.view();
    SeedIndex seeds(view);
    const int k = plan.k();
    std::vector<uint32_t> binding, cand;
    WalkScratch scratch;
    for (uint64_t i = 0; i < count; ++i) {
      CounterRng rng(seed, worker, first + i);
      CounterRng rng2(seed, worker, first + i);
      SampledCount ref = draw_sample(view, seeds, plan, rng2);
      // re-walk to capture bindings
      uint64_t work = 0;
      auto [u, v] = seeds.arc(view, rng.next_below(seeds.total_arcs()));
      if (plan.seed_ordered && u > v) std::swap(u, v);
      binding.assign({u, v});
      double alpha = plan.seed_scale(view.edge_count);
      bool hit = true;
      for (size_t si = 0; si < plan.steps.size(); ++si) {
        build_step_candidates(view, plan, si, binding, true, cand, work, scratch);
        if (cand.empty()) {
          hit = false;
          break;
        }
        alpha *= static_cast<double>(cand.size());
        uint32_t pick = cand[rng.next_below(cand.size())];
        binding.push_back(pick);
        if (plan.verify_mode == VerifyMode::Lazy) {
          uint32_t parent = binding[plan.steps[si].tree_parent];
          if (!sorted_contains(view.neighbors_of(parent), pick, work)) {
            hit = false;
            break;
          }
        }
      }
      if (hit && plan.verify_mode == VerifyMode::Lazy && !lazy_terminal_ok(view, plan, binding, work))
        hit = false;
      double value = hit ? alpha : 0.0;
      if (value != ref.value || hit != ref.hit)
        throw std::runtime_error("shim re-walk disagrees with draw_sample");
      values[i] = ref.value;
      hits[i] = ref.hit;
      if (bindings) {
        for (int p = 0; p < k; ++p)
          bindings[i * k + p] = p < static_cast<int>(binding.size()) ? binding[p] : 0xffffffffu;
      }
    }
  });
}

int ref_fixed_budget(const RefGraph* g, const char* spec, const char* induced, int mode, int sym,
                     uint64_t budget, uint64_t seed, int workers, agpm_accumulator* out) {
  return guard([&] {
    ExecutionPlan plan = plan_of(spec, induced, mode, sym);
    put_acc(run_fixed_budget(g->g.view(), plan, budget, seed, workers), out);
  });
}

int ref_ns_online(const RefGraph* g, const char* spec, const char* induced, int mode, int sym,
                  double eps, double delta, const agpm_online_policy* pol, uint64_t seed,
                  int workers, agpm_online_result* out) {
  return guard([&] {
    ExecutionPlan plan = plan_of(spec, induced, mode, sym);
    OnlinePolicy policy;
    policy.n_min = pol->n_min;
    policy.max_samples = pol->max_samples;
    policy.profiled_n_samples = pol->profiled_n_samples;
    OnlineResult r = run_ns_online(g->g.view(), plan, eps, delta, policy, seed, workers);
    std::memset(out, 0, sizeof(*out));
    put_rep(r.report, &out->report);
    put_acc(r.accumulator, &out->accumulator);
    out->windows = r.windows;
    out->work_units = r.work_units;
  });
}

// ---------------------------------------------------------------- exact / GS
int ref_exact_count(const RefGraph* g, const char* spec, const char* induced, int sym, int threads,
                    uint64_t* count, uint64_t* work) {
  return guard([&] {
    ExecutionPlan plan = plan_of(spec, induced, 0, sym);
    ExactCountResult r = exact_count(g->g.view(), plan, threads);
    *count = r.count;
    *work = r.work_units;
  });
}
// exact count on the colour-sparsified view (the GS inner call, gs_engine.cpp:67)
int ref_exact_count_colored(const RefGraph* g, const char* spec, const char* induced, uint32_t c,
                            uint64_t seed, int threads, uint64_t* count) {
  return guard([&] {
    ExecutionPlan plan = plan_of(spec, induced, 0, 1);
    ColoredCsr cc = ColoredCsr::color_vertices(g->g, c, seed);
    *count = exact_count(cc.sparsified_view(), plan, threads).count;
  });
}
int ref_brute_force(const RefGraph* g, const char* spec, const char* induced, uint64_t* out) {
  return guard([&] { *out = brute_force_count(g->g, parse_pattern_spec(spec, induced ? induced : "")); });
}
// scheme: 0 = Bernoulli edge, 1 = colour
int ref_gs_estimate(const RefGraph* g, const char* spec, const char* induced, int scheme, double p,
                    uint32_t colors, uint64_t seed, int threads, double* estimate, uint64_t* raw,
                    double* scale) {
  return guard([&] {
    ExecutionPlan plan = plan_of(spec, induced, 0, 1);
    SparsifyParams params = scheme == 0 ? SparsifyParams::bernoulli(p, seed)
                                        : SparsifyParams::color(colors, seed);
    GsEstimate e = gs_estimate(g->g, plan, params, threads);
    *estimate = e.estimate;
    *raw = e.raw_count;
    *scale = e.scale;
  });
}
int ref_choose_keep_probability(double eps, double delta, double count, double gamma, double* p,
                                int* useless, uint32_t* colors) {
  return guard([&] {
    KeepProbability kp = choose_keep_probability({eps, delta, count, gamma});
    *p = kp.p;
    *useless = kp.sparsification_useless;
    *colors = kp.color_count();
  });
}
int ref_estimate_gamma(const RefGraph* g, const char* spec, uint64_t probes, uint64_t seed,
                       int64_t budget, uint64_t* out) {
  return guard([&] {
    *out = estimate_gamma(g->g.view(), parse_pattern_spec(spec, ""), probes, seed, budget);
  });
}
int ref_count_through_edge(const RefGraph* g, const char* spec, uint32_t u, uint32_t v,
                           uint64_t* out) {
  return guard([&] {
    *out = count_matches_through_edge(g->g.view(), parse_pattern_spec(spec, ""), u, v);
  });
}

// ---------------------------------------------------------------- cost model
int ref_ns_cost_cone(const RefGraph* g, const char* spec, uint64_t n_samples, double hw,
                     double* out5) {
  return guard([&] {
    ExecutionPlan plan = plan_of(spec, "", 0, 1);
    CostCone c = ns_cost_cone(g->g.view(), plan, n_samples, hw);
    out5[0] = c.lower_slope;
    out5[1] = c.upper_slope;
    out5[2] = static_cast<double>(c.n_samples);
    out5[3] = c.lower_time;
    out5[4] = c.upper_time;
  });
}
int ref_gs_cost_estimate(const RefGraph* g, const char* spec, uint32_t colors, double hw,
                         uint64_t tri, double* out3) {
  return guard([&] {
    ExecutionPlan plan = plan_of(spec, "", 0, 1);
    GsCostEstimate e = gs_cost_estimate(g->g.view(), plan, colors, hw, tri);
    out3[0] = e.preprocess_work;
    out3[1] = e.search_work;
    out3[2] = e.total_seconds;
  });
}
int ref_fast_profile(const RefGraph* g, const char* spec, double fraction, double eps,
                     uint64_t seed, int threads, uint64_t cap, double* out6) {
  return guard([&] {
    ExecutionPlan plan = plan_of(spec, "", 0, 1);
    ProfileResult r = fast_profile(g->g, plan, fraction, eps, seed, threads, cap);
    out6[0] = r.n_samples_estimate;
    out6[1] = r.mu_prime;
    out6[2] = r.scaled_count;
    out6[3] = r.epsilon_hat_final;
    out6[4] = static_cast<double>(r.n_converged);
    out6[5] = r.reliable ? 1.0 : 0.0;
  });
}

}  // extern "C"
