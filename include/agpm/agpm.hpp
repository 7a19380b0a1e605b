// agpm/agpm.hpp — header-only C++ drop-in for the reference's sampling API.
//
// Same namespace, type names and call shapes as the reference library
// (/root/reference/proj/include/agpm/*.hpp) for the hot path, implemented
// inline over the C ABI of libagpm_b200.so (include/agpm_b200.h). A caller of
//   agpm::run_ns_online(g.view(), agpm::compile_plan(p, agpm::VerifyMode::Eager),
//                       eps, delta, agpm::OnlinePolicy{}, seed)
// relinks against libagpm_b200 and runs on the B200 unchanged. Error
// behaviour mirrors the reference: std::invalid_argument, agpm::pattern_error,
// agpm::io_error, agpm::parse_error (+ agpm::device_error for CUDA faults).
//
// Device mirrors of a CsrView are cached per (graph generation, GPU): every
// CsrGraph carries a process-unique, never-reused generation id (the reference
// documents CsrGraph / CsrView as immutable, csr_graph.hpp:19-22, 43-45), so a
// freed graph whose addresses are recycled can never alias a new one. Views
// built by hand (generation 0) are uploaded per call, never cached.
//
// `workers` / `threads` map to GPUs: with W > 1 and several visible devices,
// min(W, devices) ranks run the sharded drivers (agpm_ns_online_sharded ...),
// one host thread per GPU over an in-process communicator group. Results keep
// the workers = 1 semantics of the device path (global sample id streams), so
// they are identical for every W.
#pragma once

#include <algorithm>
#include <cstdint>
#include <exception>
#include <cstring>
#include <list>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <utility>
#include <vector>

#include "agpm_b200.h"

namespace agpm {

struct parse_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct io_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct pattern_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct device_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int status) {
  if (status == AGPM_OK) return;
  const std::string msg = agpm_last_error();
  switch (status) {
    case AGPM_E_INVALID: throw std::invalid_argument(msg);
    case AGPM_E_PATTERN: throw pattern_error(msg);
    case AGPM_E_IO: throw io_error(msg);
    case AGPM_E_PARSE: throw parse_error(msg);
    default: throw device_error(msg);
  }
}
}  // namespace detail

// ------------------------------------------------------------------ rng.hpp
// Host CounterRng with the reference's exact stream (rng.hpp:26-56).
inline uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}
inline uint64_t derive_key(uint64_t seed, uint64_t s1 = 0, uint64_t s2 = 0) {
  uint64_t h = mix64(seed + 0x9e3779b97f4a7c15ull);
  h = mix64(h ^ (s1 + 0xbf58476d1ce4e5b9ull));
  return mix64(h ^ (s2 + 0x94d049bb133111ebull));
}
class CounterRng {
 public:
  explicit CounterRng(uint64_t seed, uint64_t stream1 = 0, uint64_t stream2 = 0)
      : seed_(seed), s1_(stream1), s2_(stream2), key_(derive_key(seed, stream1, stream2)) {}
  uint64_t next_u64() {
    ctr_ += 0x9e3779b97f4a7c15ull;
    return mix64(key_ ^ ctr_);
  }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  uint64_t next_below(uint64_t n) {
    unsigned __int128 m = static_cast<unsigned __int128>(next_u64()) * n;
    auto lo = static_cast<uint64_t>(m);
    if (lo < n) {
      uint64_t t = (0 - n) % n;
      while (lo < t) {
        m = static_cast<unsigned __int128>(next_u64()) * n;
        lo = static_cast<uint64_t>(m);
      }
    }
    return static_cast<uint64_t>(m >> 64);
  }
  // stream identity (device draws regenerate the stream from it)
  uint64_t seed() const { return seed_; }
  uint64_t stream1() const { return s1_; }
  uint64_t stream2() const { return s2_; }
  bool fresh() const { return ctr_ == 0; }

 private:
  uint64_t seed_, s1_, s2_, key_;
  uint64_t ctr_ = 0;
};

// ------------------------------------------------------------------ stats.hpp
struct SampleAccumulator {
  uint64_t n = 0;
  uint64_t hits = 0;
  double sum = 0.0;
  double squared_sum = 0.0;
  void add(double value, bool hit) {
    ++n;
    if (hit) ++hits;
    sum += value;
    squared_sum += value * value;
  }
  void merge(const SampleAccumulator& o) {
    n += o.n;
    hits += o.hits;
    sum += o.sum;
    squared_sum += o.squared_sum;
  }
};

struct ConvergenceReport {
  double mu = 0.0;
  double sigma = 0.0;
  double epsilon_hat = 0.0;
  uint64_t n = 0;
  bool converged = false;
  double hit_rate = 0.0;
};

inline double norm_cdf(double z) { return agpm_norm_cdf(z); }
inline double inv_norm_cdf(double q) {
  double out = 0;
  detail::check(agpm_inv_norm_cdf(q, &out));
  return out;
}
namespace detail {
inline ConvergenceReport from_c(const agpm_report& r) {
  return {r.mu, r.sigma, r.epsilon_hat, r.n, r.converged != 0, r.hit_rate};
}
inline SampleAccumulator from_c(const agpm_accumulator& a) { return {a.n, a.hits, a.sum, a.squared_sum}; }
}  // namespace detail
inline ConvergenceReport predicted_error(const SampleAccumulator& acc, double delta) {
  agpm_accumulator a{acc.n, acc.hits, acc.sum, acc.squared_sum};
  agpm_report r{};
  detail::check(agpm_predicted_error(&a, delta, &r));
  return detail::from_c(r);
}

// ------------------------------------------------------------------ pattern.hpp / plan.hpp
enum class InducedMode { Edge, Vertex };
enum class VerifyMode { Eager, Lazy };

struct Pattern {
  std::string name;
  int vertex_count = 0;
  std::vector<std::pair<int, int>> edges;
  InducedMode induced = InducedMode::Edge;
  std::string spec;  // how the ABI rebuilds it
  int edge_count() const { return static_cast<int>(edges.size()); }
  bool is_clique() const { return edge_count() == vertex_count * (vertex_count - 1) / 2; }
};

struct PlanStep {
  int pattern_vertex = -1;
  std::vector<int> in_positions, out_positions, greater_than, less_than;
  int tree_parent = -1;
  std::vector<std::pair<int, int>> verify_edges;
};

struct ExecutionPlan {
  Pattern pattern;
  VerifyMode verify_mode = VerifyMode::Eager;
  std::vector<int> order, pos_of;
  bool seed_ordered = false;
  bool symmetry_enabled = true;
  std::vector<PlanStep> steps;
  std::vector<std::pair<int, int>> closure_edges, constraints, terminal_constraints;
  agpm_plan c{};  // the ABI image
  int k() const { return pattern.vertex_count; }
  bool is_clique() const { return pattern.is_clique(); }
  double seed_scale(uint64_t edge_count) const {
    return seed_ordered ? static_cast<double>(edge_count) : 2.0 * static_cast<double>(edge_count);
  }
  std::string scaling_rule_text() const {
    char buf[512];
    detail::check(agpm_plan_scaling_rule(&c, buf, sizeof(buf)));
    return buf;
  }
};

namespace detail {
inline std::vector<std::pair<int, int>> pairs(int n, const int32_t (*a)[2]) {
  std::vector<std::pair<int, int>> v;
  for (int i = 0; i < n; ++i) v.emplace_back(a[i][0], a[i][1]);
  return v;
}
inline ExecutionPlan from_c(const agpm_plan& c, const std::string& spec) {
  ExecutionPlan p;
  p.c = c;
  p.pattern.name = c.name;
  p.pattern.vertex_count = c.k;
  p.pattern.edges = pairs(c.n_edges, c.edges);
  p.pattern.induced = c.induced ? InducedMode::Vertex : InducedMode::Edge;
  p.pattern.spec = spec;
  p.verify_mode = c.verify_mode ? VerifyMode::Lazy : VerifyMode::Eager;
  p.order.assign(c.order, c.order + c.k);
  p.pos_of.assign(c.pos_of, c.pos_of + c.k);
  p.seed_ordered = c.seed_ordered;
  p.symmetry_enabled = c.symmetry_enabled;
  for (int s = 0; s < c.n_steps; ++s) {
    const agpm_plan_step& t = c.steps[s];
    PlanStep st;
    st.pattern_vertex = t.pattern_vertex;
    st.in_positions.assign(t.in_positions, t.in_positions + t.n_in);
    st.out_positions.assign(t.out_positions, t.out_positions + t.n_out);
    st.greater_than.assign(t.greater_than, t.greater_than + t.n_gt);
    st.less_than.assign(t.less_than, t.less_than + t.n_lt);
    st.tree_parent = t.tree_parent;
    st.verify_edges = pairs(t.n_verify, t.verify_edges);
    p.steps.push_back(std::move(st));
  }
  p.closure_edges = pairs(c.n_closure, c.closure_edges);
  p.constraints = pairs(c.n_constraints, c.constraints);
  p.terminal_constraints = pairs(c.n_terminal, c.terminal_constraints);
  return p;
}
inline const char* induced_str(InducedMode m) { return m == InducedMode::Vertex ? "vertex" : "edge"; }
}  // namespace detail

// parse_pattern_spec (pattern.cpp:130-165)
inline Pattern parse_pattern_spec(const std::string& spec, const std::string& induced_override = "") {
  agpm_plan c{};
  detail::check(agpm_plan_compile(spec.c_str(), induced_override.c_str(), 0, 1, &c));
  Pattern p = detail::from_c(c, spec).pattern;
  return p;
}
inline Pattern builtin_pattern(const std::string& name) { return parse_pattern_spec(name); }
inline std::vector<std::string> builtin_pattern_names() {
  char buf[4096];
  detail::check(agpm_builtin_pattern_names(buf, sizeof(buf)));
  std::vector<std::string> out;
  std::string cur;
  for (const char* s = buf; *s; ++s) {
    if (*s == '\n') {
      out.push_back(cur);
      cur.clear();
    } else {
      cur += *s;
    }
  }
  return out;
}
// compile_plan (plan.cpp:57-137)
inline ExecutionPlan compile_plan(const Pattern& pattern, VerifyMode mode, bool enable_symmetry = true) {
  agpm_plan c{};
  std::string spec = pattern.spec;
  if (spec.empty()) {  // a hand-built Pattern: re-express it as a custom spec (pattern.cpp:130-160)
    spec = "custom:" + std::to_string(pattern.vertex_count) + ":";
    for (size_t i = 0; i < pattern.edges.size(); ++i)
      spec += (i ? "," : "") + std::to_string(pattern.edges[i].first) + "-" + std::to_string(pattern.edges[i].second);
  }
  detail::check(agpm_plan_compile(spec.c_str(), detail::induced_str(pattern.induced),
                                  mode == VerifyMode::Lazy ? 1 : 0, enable_symmetry ? 1 : 0, &c));
  return detail::from_c(c, spec);
}

// ------------------------------------------------------------------ csr_graph.hpp
struct CsrView {
  uint32_t vertex_count = 0;
  uint64_t edge_count = 0;
  const uint64_t* begin = nullptr;
  const uint64_t* end = nullptr;
  const uint32_t* neighbors = nullptr;
  bool oriented = false;
  uint64_t generation = 0;  // owner's generation id (CsrGraph::view); 0 = hand-built view
  std::span<const uint32_t> neighbors_of(uint32_t u) const { return {neighbors + begin[u], neighbors + end[u]}; }
  uint64_t degree(uint32_t u) const { return end[u] - begin[u]; }
};

class CsrGraph {
 public:
  CsrGraph() = default;
  explicit CsrGraph(agpm_host_graph* h) : h_(h, &agpm_host_graph_free) {}
  static CsrGraph from_edges(std::vector<std::pair<uint32_t, uint32_t>> edges, uint32_t min_vertex_count = 0) {
    std::vector<uint32_t> flat;
    flat.reserve(2 * edges.size());
    for (auto [u, v] : edges) {
      flat.push_back(u);
      flat.push_back(v);
    }
    agpm_host_graph* h = nullptr;
    detail::check(agpm_host_graph_from_edges(flat.data(), edges.size(), min_vertex_count, &h));
    return CsrGraph(h);
  }
  uint32_t vertex_count() const { return info().n; }
  uint64_t edge_count() const { return info().m; }
  bool oriented() const { return info().oriented; }
  CsrView view() const {
    const uint64_t* off = nullptr;
    const uint32_t* nbr = nullptr;
    detail::check(agpm_host_graph_arrays(h_.get(), &off, &nbr));
    Info i = info();
    uint64_t gen = 0;
    detail::check(agpm_host_graph_generation(h_.get(), &gen));
    return {i.n, i.m, off, off + 1, nbr, i.oriented, gen};
  }
  agpm_host_graph* handle() const { return h_.get(); }

 private:
  struct Info {
    uint32_t n;
    uint64_t m;
    bool oriented;
  };
  Info info() const {
    uint32_t n = 0;
    uint64_t m = 0, arcs = 0, maxd = 0;
    int o = 0;
    detail::check(agpm_host_graph_info(h_.get(), &n, &m, &arcs, &o, &maxd));
    return {n, m, o != 0};
  }
  std::shared_ptr<agpm_host_graph> h_;
};

inline CsrGraph load_graph_auto(const std::string& path) {
  agpm_host_graph* h = nullptr;
  detail::check(agpm_host_graph_load(path.c_str(), &h));
  return CsrGraph(h);
}
inline CsrGraph load_binary_csr(const std::string& path) { return load_graph_auto(path); }
inline void write_binary_csr(const CsrGraph& g, const std::string& path) {
  detail::check(agpm_host_graph_write_binary(g.handle(), path.c_str()));
}
inline CsrGraph orient_by_degree(const CsrGraph& g) {
  agpm_host_graph* h = nullptr;
  detail::check(agpm_host_graph_orient_by_degree(g.handle(), &h));
  return CsrGraph(h);
}

// ------------------------------------------------------------------ ns_engine.hpp
struct SampledCount {
  double value = 0.0;
  bool hit = false;
  uint64_t work_units = 0;
};
struct OnlinePolicy {
  uint64_t n_min = 1000;
  uint64_t max_samples = 1000000000;
  uint64_t profiled_n_samples = 0;
};
struct OnlineResult {
  ConvergenceReport report;
  SampleAccumulator accumulator;
  uint64_t windows = 0;
  uint64_t work_units = 0;
};

namespace detail {
using DevRef = std::shared_ptr<agpm_graph>;

inline DevRef upload(const CsrView& g) {
  const bool plain = g.end == g.begin + 1;
  uint64_t len = 0;
  for (uint32_t u = 0; u < g.vertex_count; ++u) len = std::max(len, g.end[u]);
  agpm_graph* dev = nullptr;
  check(agpm_graph_upload(g.vertex_count, g.edge_count, g.begin, plain ? nullptr : g.end, g.neighbors, len,
                          g.oriented, nullptr, &dev));
  return DevRef(dev, &agpm_graph_free);
}

// device mirror of `g` on the current GPU: cached per (generation, device) for
// CsrGraph views (small LRU per host thread), a fresh upload for hand-built views
inline DevRef device_view(const CsrView& g) {
  if (g.generation == 0) return upload(g);
  const int dev = agpm_current_device();
  struct Entry {
    uint64_t generation;
    int device;
    DevRef ref;
  };
  thread_local std::list<Entry> cache;
  for (auto it = cache.begin(); it != cache.end(); ++it)
    if (it->generation == g.generation && it->device == dev) {
      cache.splice(cache.begin(), cache, it);
      return cache.front().ref;
    }
  DevRef ref = upload(g);
  cache.push_front({g.generation, dev, ref});
  if (cache.size() > 8) cache.pop_back();
  return ref;
}

// ranks for `workers`: min(workers, visible GPUs)
inline int gpu_ranks(int workers) {
  int n = 0;
  check(agpm_device_count(&n));
  return std::max(1, std::min(workers, n));
}

// run body(rank, comm, device view) on `ranks` GPUs, one host thread each; returns rank 0's value
template <class R, class F>
R on_ranks(const CsrView& g, int ranks, F body) {
  agpm_comm_group* grp = nullptr;
  check(agpm_comm_group_create(ranks, &grp));
  std::vector<R> out(ranks);
  std::vector<std::exception_ptr> err(ranks);
  std::vector<std::thread> pool;
  for (int r = 0; r < ranks; ++r)
    pool.emplace_back([&, r] {
      agpm_comm* c = nullptr;
      try {
        check(agpm_set_device(r));
        check(agpm_comm_init_local(grp, r, &c));
        DevRef dv = device_view(g);
        out[r] = body(c, dv.get());
      } catch (...) {
        err[r] = std::current_exception();
      }
      if (c) agpm_comm_free(c);
    });
  for (auto& t : pool) t.join();
  agpm_comm_group_free(grp);
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
  return out[0];
}
}  // namespace detail

// SeedIndex (ns_engine.hpp:23-31, ns_engine.cpp:12-23): cumulative arc index so
// a uniform seed arc is one bounded draw plus a binary search; plain and
// colour-split views alike. The device path keeps its own one-gather seed-arc
// table (csrc/device.cuh); this host index serves callers that pick arcs
// themselves and validates the view handed to draw_sample.
class SeedIndex {
 public:
  explicit SeedIndex(const CsrView& g) : prefix_(static_cast<size_t>(g.vertex_count) + 1, 0) {
    for (uint32_t u = 0; u < g.vertex_count; ++u) prefix_[u + 1] = prefix_[u] + g.degree(u);
  }
  uint64_t total_arcs() const { return prefix_.back(); }
  std::pair<uint32_t, uint32_t> arc(const CsrView& g, uint64_t index) const {
    auto it = std::upper_bound(prefix_.begin(), prefix_.end(), index);
    auto u = static_cast<uint32_t>((it - prefix_.begin()) - 1);
    return {u, g.neighbors[g.begin[u] + (index - prefix_[u])]};
  }

 private:
  std::vector<uint64_t> prefix_;
};

// draw_sample (ns_engine.cpp:92-104) for a fresh worker-0 stream CounterRng(seed, 0, id)
inline SampledCount draw_sample(const CsrView& g, const SeedIndex& seeds, const ExecutionPlan& plan,
                                CounterRng& rng) {
  if (g.edge_count == 0) throw std::invalid_argument("cannot sample from an empty graph");
  if (g.oriented) throw std::invalid_argument("sampling runs on the symmetric graph");
  if (!rng.fresh() || rng.stream1() != 0)
    throw std::invalid_argument("device draw_sample takes a fresh CounterRng(seed, 0, sample_id)");
  uint64_t arcs = 0;
  for (uint32_t u = 0; u < g.vertex_count; ++u) arcs += g.degree(u);
  if (seeds.total_arcs() != arcs) throw std::invalid_argument("seed index was built for another view");
  double v = 0.0;
  uint8_t hit = 0;
  detail::check(agpm_ns_draw(detail::device_view(g).get(), &plan.c, rng.seed(), rng.stream2(), 1, &v, &hit,
                             nullptr, nullptr));
  rng.next_u64();  // the stream is consumed, as by the reference's draw
  return {v, hit != 0, 0};
}
inline SampledCount draw_sample(const CsrView& g, const ExecutionPlan& plan, CounterRng& rng) {
  return draw_sample(g, SeedIndex(g), plan, rng);
}

// run_fixed_budget (ns_engine.cpp:142-153); streams are the workers = 1 streams
inline SampleAccumulator run_fixed_budget(const CsrView& g, const ExecutionPlan& plan, uint64_t budget,
                                          uint64_t seed, int workers = 1) {
  const int ranks = detail::gpu_ranks(workers);
  if (ranks > 1)
    return detail::on_ranks<SampleAccumulator>(g, ranks, [&](agpm_comm* c, agpm_graph* dv) {
      agpm_accumulator a{};
      detail::check(agpm_ns_fixed_budget_sharded(c, dv, &plan.c, budget, seed, &a, nullptr));
      return detail::from_c(a);
    });
  agpm_accumulator a{};
  detail::check(agpm_ns_fixed_budget(detail::device_view(g).get(), &plan.c, budget, seed, &a, nullptr));
  return detail::from_c(a);
}

inline double hit_rate_report(const CsrView& g, const ExecutionPlan& plan, uint64_t sample_budget, uint64_t seed,
                              int workers = 1) {
  SampleAccumulator acc = run_fixed_budget(g, plan, sample_budget, seed, workers);
  return static_cast<double>(acc.hits) / static_cast<double>(acc.n);
}

// run_ns_online (ns_engine.cpp:106-140), workers = 1 window semantics
inline OnlineResult run_ns_online(const CsrView& g, const ExecutionPlan& plan, double eps, double delta,
                                  const OnlinePolicy& policy, uint64_t seed, int workers = 1) {
  agpm_online_policy pol{policy.n_min, policy.max_samples, policy.profiled_n_samples};
  auto wrap = [](const agpm_online_result& r) {
    return OnlineResult{detail::from_c(r.report), detail::from_c(r.accumulator), r.windows, r.work_units};
  };
  const int ranks = detail::gpu_ranks(workers);
  if (ranks > 1)
    return detail::on_ranks<OnlineResult>(g, ranks, [&](agpm_comm* c, agpm_graph* dv) {
      agpm_online_result r{};
      detail::check(agpm_ns_online_sharded(c, dv, &plan.c, eps, delta, &pol, seed, &r, nullptr));
      return wrap(r);
    });
  agpm_online_result r{};
  detail::check(agpm_ns_online(detail::device_view(g).get(), &plan.c, eps, delta, &pol, seed, &r, nullptr));
  return wrap(r);
}

// ------------------------------------------------------------------ exact_engine.hpp
struct ExactCountResult {
  uint64_t count = 0;
  uint64_t work_units = 0;  // not a parity target (algorithm-specific); 0 here
};

// exact_count (exact_engine.cpp:66-91); `threads` maps to the device
inline ExactCountResult exact_count(const CsrView& g, const ExecutionPlan& plan, int threads = 1) {
  const int ranks = detail::gpu_ranks(threads);
  if (ranks > 1)
    return detail::on_ranks<ExactCountResult>(g, ranks, [&](agpm_comm* c, agpm_graph* dv) {
      uint64_t n = 0;
      detail::check(agpm_exact_count_sharded(c, dv, &plan.c, &n, nullptr));
      return ExactCountResult{n, 0};
    });
  uint64_t c = 0;
  detail::check(agpm_exact_count(detail::device_view(g).get(), &plan.c, &c, nullptr));
  return {c, 0};
}

// brute_force_count (exact_engine.cpp:122-133): ground-truth oracle, <= 14 vertices
inline uint64_t brute_force_count(const CsrGraph& g, const Pattern& pattern) {
  const ExecutionPlan plan = compile_plan(pattern, VerifyMode::Eager);
  const CsrView v = g.view();
  uint64_t out = 0;
  detail::check(agpm_brute_force_count(v.vertex_count, v.begin, v.end, v.neighbors, &plan.c, &out));
  return out;
}

// count_matches_through_edge (exact_engine.cpp:135-213): matches whose edge set
// contains (u, v); a work budget (candidate inspections) makes it a lower bound
inline uint64_t count_matches_through_edge(const CsrView& g, const Pattern& pattern, uint32_t u, uint32_t v,
                                           int64_t* work_budget = nullptr) {
  const ExecutionPlan plan = compile_plan(pattern, VerifyMode::Eager);
  uint64_t out = 0;
  detail::check(agpm_count_matches_through_edge_view(g.vertex_count, g.edge_count, g.begin, g.end, g.neighbors,
                                                     &plan.c, u, v, work_budget, &out));
  return out;
}

// ------------------------------------------------------------------ csr_graph.hpp / gs_engine.hpp
enum class SparsifyScheme { BernoulliEdge, Color };
struct SparsifyParams {
  SparsifyScheme scheme = SparsifyScheme::Color;
  double keep_probability = 1.0;
  uint32_t color_count = 1;
  uint64_t seed = 0;
  static SparsifyParams bernoulli(double p, uint64_t seed) { return {SparsifyScheme::BernoulliEdge, p, 1, seed}; }
  static SparsifyParams color(uint32_t c, uint64_t seed) { return {SparsifyScheme::Color, 1.0 / c, c, seed}; }
};
struct GsEstimate {
  double estimate = 0.0;
  uint64_t raw_count = 0;
  double scale = 1.0;
  SparsifyParams params;
  double preprocess_seconds = 0.0;
  double search_seconds = 0.0;
  uint64_t search_work_units = 0;
};

// gs_estimate (gs_engine.cpp:42-75)
inline GsEstimate gs_estimate(const CsrGraph& g, const ExecutionPlan& plan, const SparsifyParams& params,
                              int /*threads*/ = 1) {
  agpm_gs_result r{};
  detail::check(agpm_gs_estimate(detail::device_view(g.view()).get(), &plan.c,
                                 params.scheme == SparsifyScheme::BernoulliEdge ? 0 : 1, params.keep_probability,
                                 params.color_count, params.seed, &r, nullptr));
  return {r.estimate, r.raw_count, r.scale, params, r.preprocess_seconds, r.search_seconds, 0};
}

struct ReadKBoundInputs {
  double epsilon = 0.1;
  double delta = 0.01;
  double count_estimate = 0.0;
  double gamma_estimate = 1.0;
};
struct KeepProbability {
  double p = 1.0;
  bool sparsification_useless = false;
  uint32_t color_count() const { return count_; }
  uint32_t count_ = 1;
};

// estimate_gamma (gs_engine.cpp:179-197): max matches through `probe_edges`
// uniformly drawn arcs, a lower bound on gamma; stops once the budget is spent
inline uint64_t estimate_gamma(const CsrView& g, const Pattern& pattern, uint64_t probe_edges, uint64_t seed,
                               int64_t work_budget = 50000000) {
  const ExecutionPlan plan = compile_plan(pattern, VerifyMode::Eager);
  uint64_t out = 0;
  detail::check(agpm_estimate_gamma_view(g.vertex_count, g.edge_count, g.begin, g.end, g.neighbors, &plan.c,
                                         probe_edges, seed, work_budget, &out));
  return out;
}

// choose_keep_probability (gs_engine.cpp:24-40)
inline KeepProbability choose_keep_probability(const ReadKBoundInputs& in) {
  agpm_keep_probability k{};
  detail::check(agpm_choose_keep_probability(in.epsilon, in.delta, in.count_estimate, in.gamma_estimate, &k));
  return {k.p, k.sparsification_useless != 0, k.color_count};
}

// ------------------------------------------------------------------ colored_csr.hpp
// ColoredCsr on the device: the same-colour view (colored_csr.cpp:90-93) is a
// device graph; colours and the same-colour edge count come back to the host.
class ColoredCsr {
 public:
  static ColoredCsr color_vertices(const CsrGraph& g, uint32_t color_count, uint64_t seed) {
    ColoredCsr c(g, color_count);
    c.colors_.resize(g.vertex_count());
    agpm_graph* v = nullptr;
    detail::check(agpm_color_split(detail::device_view(g.view()).get(), color_count, seed, c.colors_.data(), &c.same_,
                                   &v, nullptr));
    c.view_.reset(v, &agpm_graph_free);
    return c;
  }
  static ColoredCsr with_colors(const CsrGraph& g, std::vector<uint32_t> colors, uint32_t color_count) {
    ColoredCsr c(g, color_count);
    c.colors_ = std::move(colors);
    agpm_graph* v = nullptr;
    detail::check(agpm_color_split_with_colors(detail::device_view(g.view()).get(), c.colors_.data(), color_count,
                                               &c.same_, &v, nullptr));
    c.view_.reset(v, &agpm_graph_free);
    return c;
  }
  // merge_colors (colored_csr.cpp:56-88)
  ColoredCsr merge_colors(const std::vector<uint32_t>& group_map) const {
    uint32_t coarse_count = 0;
    for (uint32_t gc : group_map) coarse_count = std::max(coarse_count, gc + 1);
    ColoredCsr c(base_, coarse_count);
    c.colors_.resize(base_.vertex_count());
    agpm_graph* v = nullptr;
    detail::check(agpm_merge_colors(detail::device_view(base_.view()).get(), colors_.data(), color_count_,
                                    group_map.data(), static_cast<uint32_t>(group_map.size()), c.colors_.data(),
                                    &c.same_, &v, nullptr));
    c.view_.reset(v, &agpm_graph_free);
    return c;
  }
  const std::vector<uint32_t>& colors() const { return colors_; }
  uint32_t color_count() const { return color_count_; }
  uint64_t same_color_edge_count() const { return same_; }
  // exact count on the same-colour view (the raw count gs_estimate scales)
  ExactCountResult exact_count_sparsified(const ExecutionPlan& plan) const {
    uint64_t n = 0;
    detail::check(agpm_exact_count(view_.get(), &plan.c, &n, nullptr));
    return {n, 0};
  }

 private:
  ColoredCsr(const CsrGraph& g, uint32_t c) : base_(g), color_count_(c) {}
  CsrGraph base_;
  uint32_t color_count_ = 1;
  std::vector<uint32_t> colors_;
  uint64_t same_ = 0;
  std::shared_ptr<agpm_graph> view_;
};

// ------------------------------------------------------------------ cost_model.hpp
struct CostCone {
  double lower_slope = 0.0;
  double upper_slope = 0.0;
  uint64_t n_samples = 0;
  double lower_time = 0.0;
  double upper_time = 0.0;
};
struct GsCostEstimate {
  double preprocess_work = 0.0;
  double search_work = 0.0;
  double total_seconds = 0.0;
  uint32_t color_count = 1;
};
struct ProfileResult {
  double n_samples_estimate = 0.0;
  double mu_prime = 0.0;
  double scaled_count = 0.0;
  double epsilon_hat_final = 0.0;
  uint64_t n_converged = 0;
  double fraction = 0.0;
  bool reliable = false;
  double seconds = 0.0;
};
enum class Scheme { NS, GS };

// ns_cost_cone (cost_model.cpp:78-110)
inline CostCone ns_cost_cone(const CsrView& g, const ExecutionPlan& plan, uint64_t n_samples, double hw_const) {
  uint64_t arcs = 0;
  for (uint32_t u = 0; u < g.vertex_count; ++u) arcs += g.end[u] - g.begin[u];
  agpm_cost_cone c{};
  detail::check(agpm_ns_cost_cone(g.vertex_count, static_cast<double>(arcs), &plan.c, n_samples, hw_const, &c));
  return {c.lower_slope, c.upper_slope, c.n_samples, c.lower_time, c.upper_time};
}
// gs_cost_estimate (cost_model.cpp:112-145)
inline GsCostEstimate gs_cost_estimate(const CsrView& g, const ExecutionPlan& plan, uint32_t colors, double hw_const,
                                       uint64_t triangle_count) {
  agpm_gs_cost c{};
  detail::check(agpm_gs_cost_estimate(g.vertex_count, static_cast<double>(g.edge_count), &plan.c, colors, hw_const,
                                      triangle_count, &c));
  return {c.preprocess_work, c.search_work, c.total_seconds, c.color_count};
}
// fast_profile (cost_model.cpp:147-190): Bernoulli sparsification + online NS on the device
inline ProfileResult fast_profile(const CsrGraph& g, const ExecutionPlan& plan, double profile_fraction,
                                  double user_epsilon, uint64_t seed, int /*threads*/ = 1,
                                  uint64_t profiler_sample_cap = 1000000) {
  agpm_profile_result r{};
  detail::check(agpm_fast_profile(detail::device_view(g.view()).get(), &plan.c, profile_fraction, user_epsilon, seed,
                                  profiler_sample_cap, &r, nullptr));
  return {r.n_samples_estimate, r.mu_prime, r.scaled_count, r.epsilon_hat_final, r.n_converged, r.fraction,
          r.reliable != 0, r.seconds};
}
// select_scheme (cost_model.cpp:192-194)
inline Scheme select_scheme(const CostCone& cone, const GsCostEstimate& gs) {
  const agpm_cost_cone c{cone.lower_slope, cone.upper_slope, cone.n_samples, cone.lower_time, cone.upper_time};
  const agpm_gs_cost m{gs.preprocess_work, gs.search_work, gs.total_seconds, gs.color_count};
  return agpm_select_scheme(&c, &m) == 1 ? Scheme::GS : Scheme::NS;
}

}  // namespace agpm
