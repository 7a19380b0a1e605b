// Hybrid fine/coarse scheme selection, host C++
// over the device engines:
//   choose_keep_probability        gs_engine.cpp:24-40
//   count_matches_through_edge     exact_engine.cpp:135-213  (host, budgeted backtracking)
//   estimate_gamma                 gs_engine.cpp:179-197
//   ns_model_step_work / cone      cost_model.cpp:78-110
//   gs_cost_estimate               cost_model.cpp:112-145
//   fast_profile                   cost_model.cpp:147-190   (device Bernoulli + device NS)
//   select_scheme                  cost_model.cpp:192-194
//   derive_gs_parameters + loose-mode cmd_count   agpm_main.cpp:221-287
// The reference's hardware constant is a CPU merge benchmark; both sides of
// select_scheme are (hw x work units), so the decision does not depend on it —
// the device constant (agpm_calibrate_hardware_constant) only scales reported seconds.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <functional>
#include <future>
#include <vector>

#include "common.hpp"
#include "host_graph.hpp"
#include "rng.cuh"

namespace agpm_b200 {
namespace {

constexpr double kSeedUnits = 16.0;   // cost_model.cpp:91-93
constexpr double kSampleUnits = 8.0;

double log2_ceil(double x) { return x <= 1.0 ? 1.0 : std::ceil(std::log2(x)); }

double step_work(double d, const agpm_plan& plan, int si) {  // cost_model.cpp:78-90
  const agpm_plan_step& st = plan.steps[si];
  if (plan.verify_mode == 0) {
    const double t = st.n_in;
    return (t <= 1.0 ? d : t * d) + static_cast<double>(st.n_out) * d;
  }
  return static_cast<double>(si + 2) * d + log2_ceil(d);
}

bool has_edge(const agpm_plan& p, int a, int b) { return (p.adjacency[a] >> b) & 1u; }

uint64_t automorphism_count(const agpm_plan& p) {
  std::vector<int> perm(p.k);
  for (int i = 0; i < p.k; ++i) perm[i] = i;
  uint64_t n = 0;
  do {
    bool ok = true;
    for (int e = 0; e < p.n_edges && ok; ++e)
      if (!has_edge(p, perm[p.edges[e][0]], perm[p.edges[e][1]])) ok = false;
    if (ok) ++n;
  } while (std::next_permutation(perm.begin(), perm.end()));
  return n;
}

bool sorted_contains(const uint32_t* s, uint64_t len, uint32_t x) {
  return std::binary_search(s, s + len, x);
}

}  // namespace

// A host CsrView (csr_graph.hpp:23-41): begin/end per vertex, so split views work too.
struct HostView {
  uint32_t n = 0;
  uint64_t edge_count = 0;
  const uint64_t* begin = nullptr;
  const uint64_t* end = nullptr;
  const uint32_t* nbr = nullptr;
  uint64_t degree(uint32_t x) const { return end[x] - begin[x]; }
};

HostView view_of(const HostGraph& g) {
  return {g.n, g.edge_count, g.offsets.data(), g.offsets.data() + 1, g.neighbors.data()};
}

// count_matches_through_edge (exact_engine.cpp:135-213) on a host view
uint64_t count_matches_through_edge_view(const HostView& g, const agpm_plan& p, uint32_t u, uint32_t v,
                                         int64_t* work_budget) {
  if (u >= g.n || v >= g.n) throw std::invalid_argument("edge endpoint out of range");
  const int k = p.k;
  uint64_t maps = 0;
  std::vector<uint32_t> image(k, 0);
  std::vector<int> ext_order;
  auto nb = [&](uint32_t x) { return g.nbr + g.begin[x]; };
  // The pool is scanned in ascending order, so membership of its candidates in another
  // assigned vertex's list is answered by a cursor that only moves forward (gallop, then a
  // binary search inside the last stride): the same predicate as the reference's
  // sorted_contains per candidate at a fraction of the cache misses. Injectivity is checked
  // against the <= k assigned images instead of an n-sized marker array.
  auto seek = [](const uint32_t* a, uint64_t n, uint64_t& pos, uint32_t x) {
    if (pos < n && a[pos] < x) {
      uint64_t lo = pos, step = 1;
      while (lo + step < n && a[lo + step] < x) {
        lo += step;
        step <<= 1;
      }
      uint64_t hi = std::min(lo + step, n);
      ++lo;  // a[lo - 1] < x <= a[hi] (or hi == n)
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (a[mid] < x)
          lo = mid + 1;
        else
          hi = mid;
      }
      pos = lo;
    }
    return pos < n && a[pos] == x;
  };
  std::function<uint64_t(size_t, uint32_t)> extend = [&](size_t depth, uint32_t assigned) -> uint64_t {
    if (depth == ext_order.size()) return 1;
    if (work_budget && *work_budget <= 0) return 0;
    const int pv = ext_order[depth];
    int pool_parent = -1;
    for (int prev = 0; prev < k; ++prev)
      if (((assigned >> prev) & 1u) && has_edge(p, prev, pv))
        if (pool_parent < 0 || g.degree(image[prev]) < g.degree(image[pool_parent])) pool_parent = prev;
    uint64_t total = 0;
    const uint32_t* pool = nb(image[pool_parent]);
    const uint64_t plen = g.degree(image[pool_parent]);
    if (work_budget) *work_budget -= static_cast<int64_t>(plen);
    // the other assigned vertices whose lists decide a candidate, with their cursors
    int chk[AGPM_MAX_K], nchk = 0;
    bool want[AGPM_MAX_K];
    uint64_t cur[AGPM_MAX_K];
    for (int prev = 0; prev < k; ++prev) {
      if (prev == pool_parent || !((assigned >> prev) & 1u)) continue;
      const bool w = has_edge(p, prev, pv);
      if (!w && !p.induced) continue;
      chk[nchk] = prev;
      want[nchk] = w;
      cur[nchk] = 0;
      ++nchk;
    }
    const bool last = depth + 1 == ext_order.size();
    for (uint64_t i = 0; i < plen; ++i) {
      const uint32_t cand = pool[i];
      bool ok = true;
      for (int prev = 0; prev < k && ok; ++prev)
        if (((assigned >> prev) & 1u) && image[prev] == cand) ok = false;
      for (int c = 0; c < nchk && ok; ++c)
        if (want[c] != seek(nb(image[chk[c]]), g.degree(image[chk[c]]), cur[c], cand)) ok = false;
      if (!ok) continue;
      if (last) {
        ++total;
        continue;
      }
      image[pv] = cand;
      total += extend(depth + 1, assigned | (1u << pv));
    }
    return total;
  };
  for (int e = 0; e < p.n_edges; ++e) {
    const int a = p.edges[e][0], b = p.edges[e][1];
    ext_order.clear();
    uint32_t reached = (1u << a) | (1u << b);
    while (ext_order.size() + 2 < static_cast<size_t>(k)) {
      for (int pv = 0; pv < k; ++pv) {
        if ((reached >> pv) & 1u) continue;
        bool touches = false;
        for (int prev = 0; prev < k; ++prev)
          if (((reached >> prev) & 1u) && has_edge(p, prev, pv)) touches = true;
        if (touches) {
          ext_order.push_back(pv);
          reached |= 1u << pv;
          break;
        }
      }
    }
    for (int flip = 0; flip < 2; ++flip) {
      const uint32_t da = flip ? v : u, db = flip ? u : v;
      if (!sorted_contains(nb(da), g.degree(da), db)) continue;
      image[a] = da;
      image[b] = db;
      maps += extend(0, (1u << a) | (1u << b));
    }
  }
  return maps / automorphism_count(p);
}

uint64_t count_matches_through_edge_host(const HostGraph& g, const agpm_plan& p, uint32_t u, uint32_t v,
                                         int64_t* work_budget) {
  return count_matches_through_edge_view(view_of(g), p, u, v, work_budget);
}

// estimate_gamma (gs_engine.cpp:179-197)
uint64_t estimate_gamma_view(const HostView& g, const agpm_plan& p, uint64_t probe_edges, uint64_t seed,
                             int64_t work_budget) {
  if (probe_edges < 1) throw std::invalid_argument("probe count must be >= 1");
  if (g.edge_count == 0) return 0;
  std::vector<uint64_t> prefix(static_cast<size_t>(g.n) + 1, 0);
  for (uint32_t x = 0; x < g.n; ++x) prefix[x + 1] = prefix[x] + g.degree(x);
  CounterRng rng(seed, 0x67616d6dull);  // "gamm"
  uint64_t best = 0;
  // one budget across the probes: a lower bound either way, so running out
  // mid-probe just stops with the maximum seen so far
  for (uint64_t i = 0; i < probe_edges && work_budget > 0; ++i) {
    const uint64_t idx = rng.next_below(prefix.back());
    const auto it = std::upper_bound(prefix.begin(), prefix.end(), idx);
    const auto u = static_cast<uint32_t>((it - prefix.begin()) - 1);
    const uint32_t v = g.nbr[g.begin[u] + (idx - prefix[u])];
    best = std::max(best, count_matches_through_edge_view(g, p, u, v, &work_budget));
  }
  return best;
}

uint64_t estimate_gamma_host(const HostGraph& g, const agpm_plan& p, uint64_t probe_edges, uint64_t seed,
                             int64_t work_budget) {
  return estimate_gamma_view(view_of(g), p, probe_edges, seed, work_budget);
}

}  // namespace agpm_b200

using namespace agpm_b200;

extern "C" {

int agpm_choose_keep_probability(double eps, double delta, double count_estimate, double gamma_estimate,
                                 agpm_keep_probability* out) {
  return guarded([&] {  // gs_engine.cpp:24-40
    if (!(eps > 0.0) || !(eps < 1.0)) throw std::invalid_argument("epsilon must be inside (0,1)");
    if (!(delta > 0.0) || !(delta < 1.0)) throw std::invalid_argument("delta must be inside (0,1)");
    if (gamma_estimate <= 0.0) throw std::invalid_argument("gamma estimate must be positive");
    out->p = 1.0;
    out->sparsification_useless = 0;
    if (count_estimate <= 0.0) {
      out->sparsification_useless = 1;
    } else {
      const double p = -3.0 * std::log(delta / 2.0) * gamma_estimate / (eps * eps * count_estimate);
      out->p = std::min(1.0, p);
    }
    out->color_count = out->p >= 1.0 ? 1u : std::max<uint32_t>(static_cast<uint32_t>(1.0 / out->p), 1u);
  });
}

int agpm_ns_cost_cone(double vertex_count, double arc_count, const agpm_plan* plan, uint64_t n_samples,
                      double hw_const, agpm_cost_cone* out) {
  return guarded([&] {  // cost_model.cpp:92-110
    const double d = vertex_count == 0 ? 0.0 : arc_count / vertex_count;
    double full = kSeedUnits;
    for (int si = 0; si < plan->n_steps; ++si) full += step_work(d, *plan, si) + kSampleUnits;
    if (plan->verify_mode == 1) full += static_cast<double>(plan->n_closure) * log2_ceil(d);
    double first_break = kSeedUnits;
    if (plan->n_steps > 0) first_break += step_work(d, *plan, 0);
    out->lower_slope = hw_const * first_break;
    out->upper_slope = hw_const * full;
    out->n_samples = n_samples;
    out->lower_time = out->lower_slope * static_cast<double>(n_samples);
    out->upper_time = out->upper_slope * static_cast<double>(n_samples);
  });
}

int agpm_gs_cost_estimate(double vertex_count, double edge_count, const agpm_plan* plan, uint32_t colors,
                          double hw_const, uint64_t triangle_count, agpm_gs_cost* out) {
  return guarded([&] {  // cost_model.cpp:112-145
    if (colors == 0) throw std::invalid_argument("color count must be >= 1");
    const double p = 1.0 / static_cast<double>(colors);
    const double n = vertex_count, m = edge_count, t_count = static_cast<double>(triangle_count);
    out->color_count = colors;
    out->preprocess_work = m * (1.0 + p);
    const double p1 = 2.0 * m * p / (n * n);
    const double p2 = t_count * n / (2.0 * m * m);
    const double sparse_degree = n > 0 ? 2.0 * m * p / n : 0.0;
    double below = 0.0;
    for (int idx = plan->n_steps; idx-- > 0;) {
      const agpm_plan_step& st = plan->steps[idx];
      const double t = st.n_in;
      const double op_cost = std::max(t, 1.0) * sparse_degree + static_cast<double>(st.n_out) * sparse_degree;
      const double level_size = t >= 2.0 ? n * p1 * std::pow(p2, t - 1.0) : (m * p > 0 ? n / (m * p) : 0.0);
      below = op_cost + level_size * below;
    }
    out->search_work = m * p * below;
    out->total_seconds = (out->preprocess_work + out->search_work) * hw_const;
  });
}

int agpm_select_scheme(const agpm_cost_cone* cone, const agpm_gs_cost* gs) {  // cost_model.cpp:192-194
  return gs->total_seconds < cone->lower_time ? 1 : 0;
}

int agpm_count_matches_through_edge(const agpm_host_graph* g, const agpm_plan* plan, uint32_t u, uint32_t v,
                                    uint64_t* out) {
  return guarded([&] { *out = count_matches_through_edge_host(g->g, *plan, u, v, nullptr); });
}

int agpm_estimate_gamma(const agpm_host_graph* g, const agpm_plan* plan, uint64_t probe_edges, uint64_t seed,
                        int64_t work_budget, uint64_t* out) {
  return guarded([&] { *out = estimate_gamma_host(g->g, *plan, probe_edges, seed, work_budget); });
}

int agpm_brute_force_count(uint32_t n, const uint64_t* begin, const uint64_t* end, const uint32_t* neighbors,
                           const agpm_plan* plan, uint64_t* out) {
  // exact_engine.cpp:93-133: every injective map of the pattern (vertex order
  // 0..k-1) into the graph whose mapped pattern edges are graph edges (and, in
  // the induced mode, whose non-edges are not), divided by |Aut|
  return guarded([&] {
    if (!begin || !plan || !out || (n && !neighbors)) throw std::invalid_argument("null argument");
    if (n > 14) throw std::invalid_argument("brute-force oracle is limited to 14 vertices");
    const HostView g{n, 0, begin, end ? end : begin + 1, neighbors};
    const agpm_plan& p = *plan;
    std::vector<uint32_t> image(p.k, 0);
    std::vector<bool> used(n, false);
    auto adjacent = [&](uint32_t a, uint32_t b) { return sorted_contains(g.nbr + g.begin[a], g.degree(a), b); };
    std::function<uint64_t(int)> place = [&](int pv) -> uint64_t {
      if (pv == p.k) return 1;
      uint64_t total = 0;
      for (uint32_t x = 0; x < n; ++x) {
        if (used[x]) continue;
        bool ok = true;
        for (int q = 0; q < pv && ok; ++q) {
          const bool want = has_edge(p, q, pv);
          if (!want && !p.induced) continue;
          if (want != adjacent(image[q], x)) ok = false;
        }
        if (!ok) continue;
        image[pv] = x;
        used[x] = true;
        total += place(pv + 1);
        used[x] = false;
      }
      return total;
    };
    *out = place(0) / automorphism_count(p);
  });
}

int agpm_count_matches_through_edge_view(uint32_t n, uint64_t edge_count, const uint64_t* begin,
                                         const uint64_t* end, const uint32_t* neighbors, const agpm_plan* plan,
                                         uint32_t u, uint32_t v, int64_t* work_budget, uint64_t* out) {
  return guarded([&] {
    if (!begin || !plan || !out || (n && !neighbors)) throw std::invalid_argument("null argument");
    const HostView g{n, edge_count, begin, end ? end : begin + 1, neighbors};
    *out = count_matches_through_edge_view(g, *plan, u, v, work_budget);
  });
}

int agpm_estimate_gamma_view(uint32_t n, uint64_t edge_count, const uint64_t* begin, const uint64_t* end,
                             const uint32_t* neighbors, const agpm_plan* plan, uint64_t probe_edges, uint64_t seed,
                             int64_t work_budget, uint64_t* out) {
  return guarded([&] {
    if (!begin || !plan || !out || (n && !neighbors)) throw std::invalid_argument("null argument");
    const HostView g{n, edge_count, begin, end ? end : begin + 1, neighbors};
    *out = estimate_gamma_view(g, *plan, probe_edges, seed, work_budget);
  });
}

int agpm_fast_profile(agpm_graph* g, const agpm_plan* plan, double profile_fraction, double user_epsilon,
                      uint64_t seed, uint64_t profiler_sample_cap, agpm_profile_result* out, void* stream) {
  return guarded([&] {  // cost_model.cpp:147-190 (device Bernoulli sparsify + device online NS)
    if (!(profile_fraction > 0.0) || !(profile_fraction < 1.0))
      throw std::invalid_argument("profile fraction must be inside (0,1)");
    std::memset(out, 0, sizeof(*out));
    out->fraction = profile_fraction;
    auto t0 = std::chrono::steady_clock::now();
    agpm_graph* sparse = nullptr;
    if (agpm_bernoulli_sparsify(g, profile_fraction, derive_key(seed, 0x70726f66ull, 0), &sparse, stream) != AGPM_OK)
      throw std::runtime_error(agpm_last_error());
    uint64_t ms = 0, full_m = 0, full_arcs = 0, sparse_arcs = 0;
    uint32_t n = 0;
    agpm_graph_info(sparse, &n, &ms, &sparse_arcs, nullptr, nullptr);
    agpm_graph_info(g, &n, &full_m, &full_arcs, nullptr, nullptr);
    if (ms == 0) {
      agpm_graph_free(sparse);
      return;  // unreliable
    }
    agpm_online_policy pol{1000, profiler_sample_cap, 0};
    agpm_online_result run{};
    const int st = agpm_ns_online(sparse, plan, 0.5, 0.01, &pol, seed, &run, stream);
    uint64_t dmax_full = 0, dmax_sparse = 0;
    agpm_graph_max_degree(g, &dmax_full);
    agpm_graph_max_degree(sparse, &dmax_sparse);
    agpm_graph_free(sparse);
    if (st != AGPM_OK) throw std::runtime_error(agpm_last_error());
    out->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    out->n_converged = run.report.n;
    out->mu_prime = run.report.mu;
    out->epsilon_hat_final = run.report.epsilon_hat;
    if (!run.report.converged || !(run.report.mu > 0.0)) return;  // cap hit: unreliable
    const int l = plan->n_edges, k = plan->k;
    out->scaled_count = out->mu_prime * std::pow(profile_fraction, -l);
    const double rho_ratio = (static_cast<double>(full_m) * std::pow(static_cast<double>(dmax_full), k - 2)) /
                             (static_cast<double>(ms) * std::pow(static_cast<double>(dmax_sparse), k - 2));
    const double ratio = out->epsilon_hat_final / user_epsilon;
    out->n_samples_estimate = static_cast<double>(out->n_converged) * ratio * ratio *
                              (out->mu_prime / out->scaled_count) * rho_ratio;
    if (out->n_samples_estimate < 1.0) out->n_samples_estimate = 1.0;
    out->reliable = 1;
  });
}

// loose-mode cmd_count (agpm_main.cpp:221-287): profile, gamma, keep probability,
// both cost models, select, run the chosen engine.
int agpm_count_hybrid(const agpm_host_graph* hg, agpm_graph* g, const agpm_plan* plan, double eps, double confidence,
                      uint64_t seed, double profile_fraction, double hw_const, agpm_hybrid_result* out, void* stream) {
  return guarded([&] {
    std::memset(out, 0, sizeof(*out));
    const double delta = 1.0 - confidence;
    uint32_t n = 0;
    uint64_t m = 0, arcs = 0;
    agpm_graph_info(g, &n, &m, &arcs, nullptr, nullptr);
    // gamma probing is host work on the host CSR (budgeted, sequential by definition:
    // gs_engine.cpp:179-197): it runs on its own thread while the device counts triangles
    // and profiles; the result is only used when the profile turns out reliable
    const uint64_t probes = std::min<uint64_t>(1000, std::max<uint64_t>(m, 1));
    auto gamma_job = std::async(std::launch::async, [&] {
      return m ? estimate_gamma_host(hg->g, *plan, probes, seed + 17, 50000000) : uint64_t{0};
    });
    struct Join {  // the job reads hg / plan: never let it outlive this call
      std::future<uint64_t>& f;
      ~Join() {
        if (f.valid()) f.wait();
      }
    } join{gamma_job};
    uint64_t tri = 0;
    if (agpm_triangle_count(g, &tri, stream) != AGPM_OK) throw std::runtime_error(agpm_last_error());
    if (agpm_fast_profile(g, plan, profile_fraction, eps, seed, 1000000, &out->profile, stream) != AGPM_OK)
      throw std::runtime_error(agpm_last_error());
    agpm_keep_probability keep{};
    if (!out->profile.reliable) {
      if (agpm_choose_keep_probability(eps, delta, 0.0, 1.0, &keep) != AGPM_OK) throw std::runtime_error(agpm_last_error());
      out->decision = 0;
      out->gamma = 1.0;
    } else {
      const uint64_t gm = gamma_job.get();
      out->gamma = 2.0 * static_cast<double>(std::max<uint64_t>(1, gm));  // agpm_main.cpp:230-232
      if (agpm_choose_keep_probability(eps, delta, out->profile.scaled_count, out->gamma, &keep) != AGPM_OK)
        throw std::runtime_error(agpm_last_error());
      const auto n_samples = static_cast<uint64_t>(std::max(1.0, out->profile.n_samples_estimate));
      agpm_ns_cost_cone(n, static_cast<double>(arcs), plan, n_samples, hw_const, &out->cone);
      const uint32_t model_colors = std::max<uint32_t>(2, keep.color_count);
      agpm_gs_cost_estimate(n, static_cast<double>(m), plan, model_colors, hw_const, tri, &out->gs_model);
      out->decision = agpm_select_scheme(&out->cone, &out->gs_model);
    }
    out->keep = keep;
    if (out->decision == 1) {  // run_gs_mode at the priced colour count; repeat 0 seed (agpm_main.cpp:176)
      agpm_gs_result r{};
      if (agpm_gs_estimate(g, plan, 1, 1.0, out->gs_model.color_count, derive_key(seed, 0, 0), &r, stream) != AGPM_OK)
        throw std::runtime_error(agpm_last_error());
      out->estimate = r.estimate;
      out->gs = r;
    } else {  // run_ns_mode with the profiled sample count
      agpm_online_policy pol{1000, 1000000000ull, 0};
      if (out->profile.reliable && out->profile.n_samples_estimate >= 1.0)
        pol.profiled_n_samples = static_cast<uint64_t>(out->profile.n_samples_estimate);
      if (agpm_ns_online(g, plan, eps, delta, &pol, seed, &out->ns, stream) != AGPM_OK)
        throw std::runtime_error(agpm_last_error());
      out->estimate = out->ns.report.mu;
    }
  });
}

int agpm_calibrate_hardware_constant(double* out) {
  return guarded([&] {
    // device sampler on RMAT-16 (ef 16), triangle plan: seconds per cone upper-slope work unit
    HostGraph hg = relabel_by_degree(gen_rmat(16, 16, 0.57, 0.19, 0.19, 0xca11b));
    agpm_graph* g = nullptr;
    if (agpm_graph_upload(hg.n, hg.edge_count, hg.offsets.data(), nullptr, hg.neighbors.data(), hg.neighbors.size(),
                          0, nullptr, &g) != AGPM_OK)
      throw std::runtime_error(agpm_last_error());
    agpm_plan plan{};
    agpm_plan_compile("triangle", "", 0, 1, &plan);
    agpm_accumulator acc{};
    const uint64_t budget = 1ull << 22;
    agpm_ns_fixed_budget(g, &plan, 1ull << 18, 1, &acc, nullptr);  // warm up
    auto t0 = std::chrono::steady_clock::now();
    const int st = agpm_ns_fixed_budget(g, &plan, budget, 2, &acc, nullptr);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    agpm_graph_free(g);
    if (st != AGPM_OK) throw std::runtime_error(agpm_last_error());
    agpm_cost_cone cone{};
    agpm_ns_cost_cone(hg.n, static_cast<double>(hg.offsets.back()), &plan, 1, 1.0, &cone);
    *out = secs / (static_cast<double>(budget) * cone.upper_slope);
  });
}

}  // extern "C"
