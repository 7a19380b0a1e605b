// Sampling engine host side + convergence kernels.
//
// Sampling kernels live in ns_warp.cu (warp-cooperative, default) and
// ns_lane.cu (one sample per lane, for tiny adjacency lists). This file owns
// strategy choice, the per-window moment reduction, the on-device convergence
// check and the run_fixed_budget / run_ns_online / draw_sample drivers.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include <cstdlib>

#include "comm.hpp"
#include "ns_common.cuh"
#include "stats.hpp"

namespace agpm_b200 {

// ------------------------------------------------------------ moments / convergence
// One warp per window; fixed-shape shuffle tree => deterministic partials.
__global__ void window_moments_kernel(const double* __restrict__ v, unsigned long long count,
                                      unsigned long long window, agpm_accumulator* __restrict__ out,
                                      unsigned long long nwin) {
  const int lane = threadIdx.x & 31;
  const unsigned long long w0 = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nw = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
  for (unsigned long long w = w0; w < nwin; w += nw) {
    const unsigned long long b = w * window;
    const unsigned long long e = min(count, b + window);
    unsigned long long n = 0, hits = 0;
    double s = 0.0, sq = 0.0;
    for (unsigned long long i = b + lane; i < e; i += 32) {
      const double x = v[i];
      ++n;
      hits += x != 0.0;
      s = __dadd_rn(s, x);
      sq = __dadd_rn(sq, __dmul_rn(x, x));
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      n += __shfl_xor_sync(FULL, n, d);
      hits += __shfl_xor_sync(FULL, hits, d);
      s = __dadd_rn(s, __shfl_xor_sync(FULL, s, d));
      sq = __dadd_rn(sq, __shfl_xor_sync(FULL, sq, d));
    }
    if (lane == 0) out[w] = agpm_accumulator{n, hits, s, sq};
  }
}

struct OnlineState {
  agpm_accumulator acc;
  agpm_report rep;
  unsigned long long windows;
  int stopped;
  int pad;
};

// stats.cpp:57-70 with the reference's operation order, no FMA contraction
__device__ agpm_report predicted_error_dev(const agpm_accumulator& a, double z) {
  agpm_report r;
  r.mu = 0.0;
  r.sigma = 0.0;
  r.epsilon_hat = __longlong_as_double(0x7ff0000000000000ll);
  r.n = a.n;
  r.converged = 0;
  r.hit_rate = 0.0;
  if (a.n == 0) return r;
  const double n = (double)a.n;
  r.hit_rate = __ddiv_rn((double)a.hits, n);
  r.mu = __ddiv_rn(a.sum, n);
  if (!(a.sum > 0.0) || a.n < 2) return r;
  double var = __dsub_rn(__ddiv_rn(a.squared_sum, n), __dmul_rn(r.mu, r.mu));
  if (var < 0.0) var = 0.0;
  r.sigma = __dsqrt_rn(__ddiv_rn(var, n));
  r.epsilon_hat = __ddiv_rn(__dmul_rn(z, r.sigma), r.mu);
  return r;
}

// Merge of window partials in window order (ns_engine.cpp:121-137). The running
// accumulator is the reference's left fold (one thread adds the windows of a
// 256-window chunk in order, exactly as before); the per-window stop tests —
// a division, a square root and two more divisions each, the slow part —
// run one window per thread, and the first window that stops wins. Same sums,
// same reports, same stop window as the one-thread loop.
constexpr int kConvergeThreads = 256;
__global__ void __launch_bounds__(kConvergeThreads) converge_kernel(const agpm_accumulator* __restrict__ win,
                                                                    unsigned long long nwin, OnlineState* st,
                                                                    double z, double eps,
                                                                    unsigned long long max_samples) {
  __shared__ agpm_accumulator pre[kConvergeThreads];
  __shared__ agpm_accumulator chunk[kConvergeThreads];
  __shared__ int first;
  const int t = threadIdx.x;
  OnlineState s = *st;
  for (unsigned long long w0 = 0; w0 < nwin && !s.stopped; w0 += kConvergeThreads) {
    const int cnt = (int)min((unsigned long long)kConvergeThreads, nwin - w0);
    if (t < cnt) chunk[t] = win[w0 + t];
    if (t == 0) first = kConvergeThreads;
    __syncthreads();
    if (t == 0) {  // the left fold, in window order
      agpm_accumulator acc = s.acc;
      for (int i = 0; i < cnt; ++i) {
        acc.n += chunk[i].n;
        acc.hits += chunk[i].hits;
        acc.sum = __dadd_rn(acc.sum, chunk[i].sum);
        acc.squared_sum = __dadd_rn(acc.squared_sum, chunk[i].squared_sum);
        pre[i] = acc;
      }
    }
    __syncthreads();
    if (t < cnt) {
      const agpm_report r = predicted_error_dev(pre[t], z);
      if (r.epsilon_hat <= eps || pre[t].n >= max_samples) atomicMin(&first, t);
    }
    __syncthreads();
    const int stop = first;
    const int last = stop < cnt ? stop : cnt - 1;
    s.acc = pre[last];
    s.windows += (unsigned long long)last + 1;
    s.rep = predicted_error_dev(s.acc, z);
    if (stop < cnt) {
      if (s.rep.epsilon_hat <= eps) s.rep.converged = 1;
      s.stopped = 1;
    }
    __syncthreads();  // chunk / pre / first are rewritten by the next chunk
  }
  if (t == 0) *st = s;
}

// ------------------------------------------------------------ host side
namespace {

DevPlan make_dev_plan(const agpm_graph* g, const agpm_plan* plan) {
  if (!plan) throw std::invalid_argument("null plan");
  if (plan->k < 2 || plan->k > AGPM_MAX_K || plan->n_steps != plan->k - 2)
    throw std::invalid_argument("malformed plan");
  if (plan->verify_mode != 0 && plan->verify_mode != 1) throw std::invalid_argument("unknown verify mode");
  if (g->edge_count == 0) throw std::invalid_argument("cannot sample from an empty graph");
  if (g->oriented) throw std::invalid_argument("sampling runs on the symmetric graph");
  DevPlan d{};
  d.k = plan->k;
  d.n_steps = plan->n_steps;
  d.seed_ordered = plan->seed_ordered;
  d.alpha0 = plan->seed_ordered ? static_cast<double>(g->edge_count) : 2.0 * static_cast<double>(g->edge_count);
  for (int s = 0; s < plan->n_steps; ++s) {
    const agpm_plan_step& st = plan->steps[s];
    unsigned in = 0, out = 0, gt = 0, lt = 0;
    for (int i = 0; i < st.n_in; ++i) in |= 1u << st.in_positions[i];
    for (int i = 0; i < st.n_out; ++i) out |= 1u << st.out_positions[i];
    for (int i = 0; i < st.n_gt; ++i) gt |= 1u << st.greater_than[i];
    for (int i = 0; i < st.n_lt; ++i) lt |= 1u << st.less_than[i];
    if (in == 0 || (in >> (s + 2)) || (out >> (s + 2)) || (gt >> (s + 2)) || (lt >> (s + 2)))
      throw std::invalid_argument("malformed plan step");
    d.in_mask[s] = (unsigned short)in;
    d.out_mask[s] = (unsigned short)out;
    d.gt_mask[s] = (unsigned short)gt;
    d.lt_mask[s] = (unsigned short)lt;
    if (st.tree_parent < 0 || st.tree_parent >= s + 2) {
      if (plan->verify_mode == 1) throw std::invalid_argument("malformed plan step");
    } else {
      d.tree_parent[s] = (unsigned char)st.tree_parent;
    }
  }
  for (int s = 0; s < d.n_steps; ++s)
    for (int s2 = s + 1; s2 < d.n_steps; ++s2)
      if (((d.in_mask[s2] >> (s + 2)) & 1u) && ((d.gt_mask[s2] | d.lt_mask[s2]) & d.in_mask[s]))
        d.twin_hint[s] = 1;
  d.lazy = plan->verify_mode == 1;
  if (d.lazy) {  // pattern vertices -> positions (walker.hpp:88-107)
    auto pos = [&](int v) {
      if (v < 0 || v >= plan->k) throw std::invalid_argument("malformed plan");
      return (unsigned char)plan->pos_of[v];
    };
    if (plan->n_closure < 0 || plan->n_closure > AGPM_MAX_PAIRS || plan->n_terminal < 0 ||
        plan->n_terminal > AGPM_MAX_PAIRS)
      throw std::invalid_argument("malformed plan");
    for (int i = 0; i < plan->n_closure; ++i) {
      d.closure[i][0] = pos(plan->closure_edges[i][0]);
      d.closure[i][1] = pos(plan->closure_edges[i][1]);
    }
    d.n_closure = (unsigned char)plan->n_closure;
    for (int i = 0; i < plan->n_terminal; ++i) {
      d.terminal[i][0] = pos(plan->terminal_constraints[i][0]);
      d.terminal[i][1] = pos(plan->terminal_constraints[i][1]);
    }
    d.n_terminal = (unsigned char)plan->n_terminal;
    int na = 0;
    if (plan->induced)
      for (int a = 0; a < plan->k; ++a)
        for (int b = a + 1; b < plan->k; ++b)
          if (!((plan->adjacency[a] >> b) & 1u)) {
            d.nonadj[na][0] = pos(a);
            d.nonadj[na][1] = pos(b);
            ++na;
          }
    d.n_nonadj = (unsigned char)na;
  }
  return d;
}

GraphArgs graph_args(const agpm_graph* g) {
  GraphArgs a;
  a.vtx = g->vtx;
  a.nbr = g->nbr;
  a.seed_arcs = g->seed_arcs;
  a.arcs = g->arcs;
  a.plain = g->plain;
  a.loop_free = g->loop_free;
  a.core = g->core;
  a.core_base = g->core_base;
  a.core_wpr = g->core_wpr;
  a.twin = g->twin;
  a.n = g->n;
  return a;
}

// Strategy: one warp per sample (coalesced chunk intersections, k-ary
// searches) unless adjacency lists are tiny, where one lane per sample keeps
// 32 samples in flight per warp. Override with agpm_ns_set_strategy().
// (4 was the fused sampler: measured slower than flat and frontier everywhere, removed)
constexpr int kStrategyAuto = 0, kStrategyWarp = 1, kStrategyLane = 2, kStrategyFrontier = 3, kStrategyFlat = 5;
std::atomic<int> g_strategy{kStrategyAuto};  // process-wide setting, read once per launch

// Plans whose multi-list steps all sit in the dense core go to the flat sampler
// on graphs up to 2^26 vertices: no out-lists and a lower bound above both seed
// vertices (steps with up to three other lists run in the flat fast class, wider
// ones per element against the same core rows). Seeds are arc-uniform, hence degree-biased towards the
// hubs at the top of a relabelled graph, so such drivers are short suffixes
// inside the core. That covers the clique plans up to the 5-clique's last step
// and the 4-cycle (S_3 = N(v0) & N(v2) above v1; v2, the owner of one list, may
// lie inside [lo, hi) but is never in its own list on a loop-free view).
// Per 2^24 samples, flat vs frontier: 4-clique RMAT-20 5.8 vs 12.5 ms, RMAT-22 8.6 vs
// 14.9, RMAT-24 13.1 vs 18.1, RMAT-26 (512 K core) 22.3 vs 24.3, RMAT-27 31.6 vs 28.0; 5-clique
// RMAT-24 17.3 vs 24.8; 4-cycle RMAT-20 5.5 vs 8.8, RMAT-22 7.5 vs 11.4, RMAT-24 12.0
// vs 14.2, RMAT-25 15.9 vs 17.9. Plans without such bounds (house 144 vs 76 ms,
// dumbbell 35 vs 25, 5-path 8.9 vs 4.0) or with out-lists (4motif-cycle 295 vs 171)
// and bigger graphs stay on the frontier phases.
bool core_suffix_plan(const DevPlan& p) {
  bool multi = false;
  for (int s = 0; s < p.k - 2; ++s) {
    const int n_in = __builtin_popcount(p.in_mask[s]);
    if (n_in == 1 && p.out_mask[s] == 0) continue;  // single-list step: index arithmetic
    multi = true;
    if (p.out_mask[s] != 0 || (p.gt_mask[s] & 3u) != 3u) return false;
  }
  return multi;
}

int choose_strategy(const agpm_graph* g, const DevPlan& p, uint64_t count, int forced) {
  if (forced != kStrategyAuto) return forced;
  const uint64_t core = core_dim_setting();
  if (count >= (1ull << 18) && core_suffix_plan(p) && core && g->n <= (1u << 26)) return kStrategyFlat;
  const double avg_deg = g->n ? static_cast<double>(g->arcs) / g->n : 0.0;
  if (avg_deg <= 24.0 && g->max_degree <= 256) return kStrategyLane;
  return count >= (1ull << 18) ? kStrategyFrontier : kStrategyWarp;
}

// per-sample stream: 0 = CounterRng(seed, 0, id) (the reference's stream, the
// parity policy), 1 = Philox4x32-10 keyed by seed, counter (draw, id) — flat sampler
std::atomic<int> g_rng_policy{0};

// enqueue one sampling launch for ids [first, first+count) into d_values
void enqueue_sample(const agpm_graph* g, const DevPlan& dp, uint64_t seed, uint64_t first, uint64_t count,
                    double* d_values, uint32_t* d_bindings, unsigned long long* d_bytes, cudaStream_t s) {
  DeviceCtx& ctx = ctx_for_current_device();
  auto* cursor = static_cast<unsigned long long*>(ctx.get(0, 64));
  AGPM_CUDA(cudaMemsetAsync(cursor, 0, sizeof(unsigned long long), s));
  if (dp.k < 3 || dp.k > AGPM_MAX_K) throw std::invalid_argument("device sampler needs 3 <= k <= 9");
  const int forced = g_strategy.load(std::memory_order_relaxed);
  if (g_rng_policy.load(std::memory_order_relaxed) == 1) {  // Philox stream: the flat sampler, eager plans
    if (dp.lazy || d_bytes) throw std::invalid_argument("the Philox stream runs on the eager flat sampler");
    if (forced != kStrategyAuto && forced != kStrategyFlat)
      throw std::invalid_argument("the Philox stream runs on the flat sampler (strategy auto or flat)");
    ensure_core_bits(const_cast<agpm_graph*>(g), s);
    SampleLaunch L{graph_args(g), dp, seed, first, count, d_values, d_bindings, cursor, nullptr};
    launch_ns_flat(L, s, true);
    return;
  }
  if (dp.lazy) {  // NS-base: one warp per sample streams the union of the bound lists
    if (d_bytes) throw std::invalid_argument("the B_min sector model is defined for eager plans");
    SampleLaunch L{graph_args(g), dp, seed, first, count, d_values, d_bindings, cursor, nullptr};
    launch_ns_lazy(L, s);
    return;
  }
  const int strat = d_bytes ? kStrategyWarp : choose_strategy(g, dp, count, forced);  // B_min replay: warp kernel
  if (strat == kStrategyFrontier || strat == kStrategyFlat) ensure_core_bits(const_cast<agpm_graph*>(g), s);
  // The twin-arc index (4 B per arc, one binary search per arc to build: 1.0 ms on
  // RMAT-20, 0.94 s on RMAT-27) hints both seed lists and saves 25-120 ps per sample,
  // so it pays for itself after about as many samples as the view has arcs: it is
  // built once that many ids have been sampled on the view (same samples with or
  // without it; agpm_graph_prepare builds it at once). A one-shot online run on a
  // big graph (config 5: 1.3 M samples, 4.2 G arcs) never pays the build.
  if (strat == kStrategyFrontier || strat == kStrategyFlat) {
    auto* gm = const_cast<agpm_graph*>(g);
    if (gm->samples_drawn.fetch_add(count, std::memory_order_relaxed) >= g->arcs) ensure_twin_arcs(gm, s);
  }
  SampleLaunch L{graph_args(g), dp, seed, first, count, d_values, d_bindings, cursor, d_bytes};
  if (strat == kStrategyLane)
    launch_ns_lane(L, s);
  else if (strat == kStrategyFrontier)
    launch_ns_frontier(L, s);
  else if (strat == kStrategyFlat)
    launch_ns_flat(L, s);
  else
    launch_ns_warp(L, s);
}

void enqueue_moments(const double* d_values, uint64_t count, uint64_t window, agpm_accumulator* d_out,
                     cudaStream_t s) {
  DeviceCtx& ctx = ctx_for_current_device();
  const uint64_t nwin = (count + window - 1) / window;
  if (nwin == 0) return;
  uint64_t blocks = std::min<uint64_t>((nwin + 7) / 8, (uint64_t)ctx.sm_count * 8);
  window_moments_kernel<<<(unsigned)blocks, 256, 0, s>>>(d_values, count, window, d_out, nwin);
  count_launch();
  AGPM_CUDA(cudaGetLastError());
}

constexpr uint64_t kChunk = 1ull << 24;

// ids [lo, hi) folded into one accumulator: 2^24-sample launches, 4096-sample
// window partials (fixed shuffle trees) summed on the host in id order
agpm_accumulator fixed_budget_range(const agpm_graph* g, const DevPlan& dp, uint64_t lo, uint64_t hi, uint64_t seed,
                                    cudaStream_t s) {
  agpm_accumulator acc{0, 0, 0.0, 0.0};
  if (hi <= lo) return acc;
  DeviceCtx& ctx = ctx_for_current_device();
  const uint64_t chunk = std::min<uint64_t>(hi - lo, kChunk);
  constexpr uint64_t kWin = 4096;
  const uint64_t nwin_chunk = (chunk + kWin - 1) / kWin;
  auto* d_values = static_cast<double*>(ctx.get(1, sizeof(double) * chunk));
  auto* d_win = static_cast<agpm_accumulator*>(ctx.get(4, sizeof(agpm_accumulator) * nwin_chunk));
  auto* h_win = static_cast<agpm_accumulator*>(ctx.get_pinned(0, sizeof(agpm_accumulator) * nwin_chunk));
  for (uint64_t done = lo; done < hi; done += chunk) {
    const uint64_t c = std::min(chunk, hi - done);
    const uint64_t nw = (c + kWin - 1) / kWin;
    enqueue_sample(g, dp, seed, done, c, d_values, nullptr, nullptr, s);
    enqueue_moments(d_values, c, kWin, d_win, s);
    AGPM_CUDA(cudaMemcpyAsync(h_win, d_win, sizeof(agpm_accumulator) * nw, cudaMemcpyDeviceToHost, s));
    AGPM_CUDA(cudaStreamSynchronize(s));
    for (uint64_t w = 0; w < nw; ++w) {
      acc.n += h_win[w].n;
      acc.hits += h_win[w].hits;
      acc.sum += h_win[w].sum;
      acc.squared_sum += h_win[w].squared_sum;
    }
  }
  return acc;
}

// One round of the sharded online loop: the ids [launched, launched + round)
// of this round (round = min(world * batch, max_samples - launched)) are dealt
// to the ranks in contiguous blocks of `batch` (a multiple of the window), so
// the gathered window records are in id order and the valid ones form a prefix.
void shard_round(uint64_t launched, uint64_t batch, uint64_t window, uint64_t max_samples, int rank, int world,
                 agpm_shard_round* out) {
  const uint64_t round = std::min(batch * (uint64_t)world, max_samples - launched);
  const uint64_t lo = std::min(round, batch * (uint64_t)rank);
  out->round_ids = round;
  out->first_id = launched + lo;
  out->count = std::min(round - lo, batch);
  out->valid_windows = (round + window - 1) / window;
  out->windows_per_rank = batch / window;
}

// The online loop (ns_engine.cpp:106-140, workers = 1 semantics) on one GPU
// (c == nullptr) or over the ranks of c. Each round every rank draws its block
// of B ids (B a multiple of the window W), folds it into W-sample window
// records, the records are all-gathered in rank = id order, and every rank
// runs converge_kernel over the same records: the per-window stop test of the
// reference, so the stop n does not depend on B or on the rank count.
void online_loop(agpm_comm* c, agpm_graph* g, const agpm_plan* plan, double eps, double delta,
                 const agpm_online_policy* policy, uint64_t seed, agpm_online_result* out, void* stream) {
  if (!(eps > 0.0) || !(eps < 1.0)) throw std::invalid_argument("error bound must be inside (0,1)");
  if (!(delta > 0.0) || !(delta < 1.0)) throw std::invalid_argument("delta must be inside (0,1)");
  if (!g || !out) throw std::invalid_argument("null argument");
  DeviceGuard guard(g->device);
  const DevPlan dp = make_dev_plan(g, plan);
  agpm_online_policy pol = policy ? *policy : agpm_online_policy{1000, 1000000000ull, 0};
  DeviceCtx& ctx = ctx_for_current_device();
  cudaStream_t s = pick_stream(stream);
  const int rank = c ? comm_rank(c) : 0, world = c ? comm_world(c) : 1;
  const double z = inv_norm_cdf(1.0 - delta / 2.0);
  uint64_t window = std::max<uint64_t>(pol.n_min, 10);
  if (pol.profiled_n_samples > 0) window = std::max(window, pol.profiled_n_samples / 10);
  const uint64_t max_batch = std::max<uint64_t>(window, (kChunk / window) * window);
  // first speculative round 2^19 samples over all ranks (then doubling): one
  // pass covers most 1 %@95 % runs on config-2-sized graphs; measured time to
  // converge for 4-clique 2.04 ms (2^16 first) -> 0.80 ms (2^19), tools/ttc_probe.py
  uint64_t batch = std::min(max_batch, std::max<uint64_t>(window, ((1ull << 19) / world / window) * window));
  const uint64_t nw_max = max_batch / window;

  auto* d_values = static_cast<double*>(ctx.get(1, sizeof(double) * max_batch));
  auto* d_win = static_cast<agpm_accumulator*>(ctx.get(4, sizeof(agpm_accumulator) * (nw_max + 1)));
  agpm_accumulator* d_all = d_win;
  if (world > 1) d_all = static_cast<agpm_accumulator*>(ctx.get(6, sizeof(agpm_accumulator) * nw_max * world));
  auto* d_state = static_cast<OnlineState*>(ctx.get(5, sizeof(OnlineState)));
  auto* h_state = static_cast<OnlineState*>(ctx.get_pinned(1, sizeof(OnlineState)));
  AGPM_CUDA(cudaMemsetAsync(d_state, 0, sizeof(OnlineState), s));
  if (c) comm_barrier(c, s);
  auto t0 = std::chrono::steady_clock::now();
  uint64_t launched = 0;
  std::memset(h_state, 0, sizeof(OnlineState));
  while (launched < pol.max_samples) {
    agpm_shard_round sr{};
    shard_round(launched, batch, window, pol.max_samples, rank, world, &sr);
    const uint64_t round = sr.round_ids, mine = sr.count, nw_round = sr.valid_windows;
    if (mine) {
      enqueue_sample(g, dp, seed, sr.first_id, mine, d_values, nullptr, nullptr, s);
      enqueue_moments(d_values, mine, window, d_win, s);
    }
    if (world > 1) {
      const uint64_t nw_rank = batch / window, nw_mine = (mine + window - 1) / window;
      if (nw_mine < nw_rank)  // padding records past the cap (never reached by the stop test)
        AGPM_CUDA(cudaMemsetAsync(d_win + nw_mine, 0, sizeof(agpm_accumulator) * (nw_rank - nw_mine), s));
      comm_all_gather(c, d_win, d_all, sizeof(agpm_accumulator) * nw_rank, s);
    }
    converge_kernel<<<1, kConvergeThreads, 0, s>>>(d_all, nw_round, d_state, z, eps, pol.max_samples);
    count_launch();
    AGPM_CUDA(cudaGetLastError());
    AGPM_CUDA(cudaMemcpyAsync(h_state, d_state, sizeof(OnlineState), cudaMemcpyDeviceToHost, s));
    AGPM_CUDA(cudaStreamSynchronize(s));
    launched += round;
    if (h_state->stopped) break;
    batch = std::min(max_batch, batch * 2);
  }
  auto t1 = std::chrono::steady_clock::now();
  std::memset(out, 0, sizeof(*out));
  out->report = h_state->rep;
  out->accumulator = h_state->acc;
  out->windows = h_state->windows;
  out->samples_launched = launched;
  out->seconds = std::chrono::duration<double>(t1 - t0).count();
}

}  // namespace

}  // namespace agpm_b200

using namespace agpm_b200;

extern "C" {

int agpm_ns_set_strategy(int strategy) {
  return guarded([&] {
    if (strategy < 0 || strategy > 5 || strategy == 4)
      throw std::invalid_argument("strategy must be 0 (auto), 1 (warp), 2 (lane), 3 (frontier) or 5 (flat)");
    g_strategy = strategy;
  });
}

int agpm_ns_set_rng(int policy) {
  return guarded([&] {
    if (policy != 0 && policy != 1) throw std::invalid_argument("rng policy must be 0 (CounterRng) or 1 (Philox4x32-10)");
    g_rng_policy = policy;
  });
}

int agpm_ns_strategy_for(const agpm_graph* g, const agpm_plan* plan, uint64_t count, int* out_strategy) {
  return guarded([&] {
    if (!g || !plan || !out_strategy) throw std::invalid_argument("null argument");
    const DevPlan dp = make_dev_plan(g, plan);
    *out_strategy = choose_strategy(g, dp, count, g_strategy.load(std::memory_order_relaxed));
  });
}

int agpm_ns_set_frontier_reuse(int on) {
  return guarded([&] { set_frontier_reuse(on != 0); });
}

int agpm_ns_sample_dev(agpm_graph* g, const agpm_plan* plan, uint64_t seed, uint64_t first_id,
                       uint64_t count, double* d_values, void* stream) {
  return guarded([&] {
    const DevPlan dp = make_dev_plan(g, plan);
    if (count) enqueue_sample(g, dp, seed, first_id, count, d_values, nullptr, nullptr, pick_stream(stream));
  });
}

int agpm_window_moments_dev(const double* d_values, uint64_t count, uint64_t window,
                            agpm_accumulator* d_out, void* stream) {
  return guarded([&] {
    if (window == 0) throw std::invalid_argument("window must be >= 1");
    enqueue_moments(d_values, count, window, d_out, pick_stream(stream));
  });
}

int agpm_ns_draw(agpm_graph* g, const agpm_plan* plan, uint64_t seed, uint64_t first_id, uint64_t count,
                 double* values, uint8_t* hits, uint32_t* bindings, void* stream) {
  return guarded([&] {
    const DevPlan dp = make_dev_plan(g, plan);
    DeviceCtx& ctx = ctx_for_current_device();
    cudaStream_t s = pick_stream(stream);
    const uint64_t chunk = std::min<uint64_t>(count ? count : 1, kChunk);
    auto* d_values = static_cast<double*>(ctx.get(1, sizeof(double) * chunk));
    uint32_t* d_bind = bindings ? static_cast<uint32_t*>(ctx.get(2, sizeof(uint32_t) * chunk * dp.k)) : nullptr;
    for (uint64_t done = 0; done < count; done += chunk) {
      const uint64_t c = std::min(chunk, count - done);
      enqueue_sample(g, dp, seed, first_id + done, c, d_values, d_bind, nullptr, s);
      AGPM_CUDA(cudaMemcpyAsync(values + done, d_values, sizeof(double) * c, cudaMemcpyDeviceToHost, s));
      if (bindings)
        AGPM_CUDA(cudaMemcpyAsync(bindings + done * dp.k, d_bind, sizeof(uint32_t) * c * dp.k,
                                  cudaMemcpyDeviceToHost, s));
      AGPM_CUDA(cudaStreamSynchronize(s));
      if (hits)
        for (uint64_t i = 0; i < c; ++i) hits[done + i] = values[done + i] != 0.0;
    }
  });
}

int agpm_ns_bmin_bytes(agpm_graph* g, const agpm_plan* plan, uint64_t seed, uint64_t first_id,
                       uint64_t count, uint64_t* total_bytes, void* stream) {
  return guarded([&] {
    const DevPlan dp = make_dev_plan(g, plan);
    DeviceCtx& ctx = ctx_for_current_device();
    cudaStream_t s = pick_stream(stream);
    const uint64_t chunk = std::min<uint64_t>(count ? count : 1, kChunk);
    auto* d_values = static_cast<double*>(ctx.get(1, sizeof(double) * chunk));
    auto* d_bytes = static_cast<unsigned long long*>(ctx.get(3, 64));
    AGPM_CUDA(cudaMemsetAsync(d_bytes, 0, 8, s));
    for (uint64_t done = 0; done < count; done += chunk) {
      const uint64_t c = std::min(chunk, count - done);
      enqueue_sample(g, dp, seed, first_id + done, c, d_values, nullptr, d_bytes, s);
    }
    unsigned long long h = 0;
    AGPM_CUDA(cudaMemcpyAsync(&h, d_bytes, 8, cudaMemcpyDeviceToHost, s));
    AGPM_CUDA(cudaStreamSynchronize(s));
    *total_bytes = h;
  });
}

int agpm_ns_fixed_budget(agpm_graph* g, const agpm_plan* plan, uint64_t budget, uint64_t seed,
                         agpm_accumulator* out, void* stream) {
  // run_fixed_budget (ns_engine.cpp:142-153): one window of `budget` samples
  return guarded([&] {
    if (budget < 1) throw std::invalid_argument("sample budget must be >= 1");
    if (!g || !out) throw std::invalid_argument("null argument");
    DeviceGuard guard(g->device);
    const DevPlan dp = make_dev_plan(g, plan);
    *out = fixed_budget_range(g, dp, 0, budget, seed, pick_stream(stream));
  });
}

int agpm_ns_online(agpm_graph* g, const agpm_plan* plan, double eps, double delta,
                   const agpm_online_policy* policy, uint64_t seed, agpm_online_result* out,
                   void* stream) {
  // run_ns_online (ns_engine.cpp:106-140) with workers = 1: windows of
  // W = max(n_min, 10) (or >= profiled/10) samples; convergence is evaluated
  // after EVERY window even though the device draws speculative batches of
  // many windows, so the stop n equals the reference's.
  return guarded([&] { online_loop(nullptr, g, plan, eps, delta, policy, seed, out, stream); });
}

int agpm_ns_shard_round(uint64_t launched, uint64_t batch, uint64_t window, uint64_t max_samples, int rank,
                        int world, agpm_shard_round* out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null argument");
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("rank must be in [0, world)");
    if (window == 0 || batch == 0 || batch % window) throw std::invalid_argument("batch must be a positive multiple of the window");
    if (launched > max_samples) throw std::invalid_argument("launched past max_samples");
    shard_round(launched, batch, window, max_samples, rank, world, out);
  });
}

int agpm_ns_online_sharded(agpm_comm* c, agpm_graph* g, const agpm_plan* plan, double eps, double delta,
                           const agpm_online_policy* policy, uint64_t seed, agpm_online_result* out,
                           void* stream) {
  return guarded([&] {
    if (!c) throw std::invalid_argument("null communicator");
    online_loop(c, g, plan, eps, delta, policy, seed, out, stream);
  });
}

int agpm_ns_fixed_budget_sharded(agpm_comm* c, agpm_graph* g, const agpm_plan* plan, uint64_t budget,
                                 uint64_t seed, agpm_accumulator* out, void* stream) {
  // run_fixed_budget (ns_engine.cpp:142-153) with the ids [0, budget) split into
  // `world` contiguous shares; the ranks' accumulators are gathered and folded in
  // rank order (the reference merges its workers' accumulators in worker order)
  return guarded([&] {
    if (!c || !g || !out) throw std::invalid_argument("null argument");
    if (budget < 1) throw std::invalid_argument("sample budget must be >= 1");
    DeviceGuard guard(g->device);
    const DevPlan dp = make_dev_plan(g, plan);
    DeviceCtx& ctx = ctx_for_current_device();
    cudaStream_t s = pick_stream(stream);
    const int rank = comm_rank(c), world = comm_world(c);
    const uint64_t share = (budget + world - 1) / world;
    const uint64_t lo = std::min(budget, share * rank), hi = std::min(budget, lo + share);
    const agpm_accumulator mine = fixed_budget_range(g, dp, lo, hi, seed, s);
    auto* d = static_cast<agpm_accumulator*>(ctx.get(10, sizeof(agpm_accumulator) * (world + 1)));
    AGPM_CUDA(cudaMemcpyAsync(d + world, &mine, sizeof(mine), cudaMemcpyHostToDevice, s));
    comm_all_gather(c, d + world, d, sizeof(agpm_accumulator), s);
    std::vector<agpm_accumulator> all(world);
    AGPM_CUDA(cudaMemcpyAsync(all.data(), d, sizeof(agpm_accumulator) * world, cudaMemcpyDeviceToHost, s));
    AGPM_CUDA(cudaStreamSynchronize(s));
    agpm_accumulator acc{0, 0, 0.0, 0.0};
    for (const auto& a : all) {
      acc.n += a.n;
      acc.hits += a.hits;
      acc.sum += a.sum;
      acc.squared_sum += a.squared_sum;
    }
    *out = acc;
  });
}

}  // extern "C"
