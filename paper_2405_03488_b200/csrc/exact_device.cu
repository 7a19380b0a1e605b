// Exact subgraph counting on the device:
// exact_count / search_from_seed (exact_engine.cpp:19-91), GraphZero-style.
//
// One warp per seed arc (claimed 32 at a time), warp-uniform depth-first
// search over the plan's steps. Each level's candidate set
//   S_j = (∩ in-lists) ∩ [lo, hi) \ (∪ out-lists) \ bound vertices
// (walker.hpp:30-83; bounds skipped for oriented cliques, exact_engine.cpp:67-72)
// is built 32 driver elements at a time: each lane tests its element against
// the other lists with a splitter + shuffle + short search (as the frontier
// sampler), one ballot gives the survivors, and a popcount prefix compacts
// them into the warp's level buffer. The last eager level is only counted
// (count += |S_last|, exact_engine.cpp:34-37). Counts are exact integers.
#include <algorithm>
#include <stdexcept>

#include "ns_common.cuh"

namespace agpm_b200 {
namespace {

constexpr uint32_t INF = 0xffffffffu;

__device__ __forceinline__ uint32_t lb_seq(const uint32_t* base, uint32_t lo, uint32_t hi, uint32_t x) {
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (ldn(base, mid) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// lower_bound of x in base[lo, hi] (answer in [lo, hi]); warp-uniform, 32 probes per round
__device__ __forceinline__ uint32_t kary(const uint32_t* base, uint32_t lo, uint32_t hi, uint32_t x, int lane) {
  while (hi - lo > 32) {
    const uint32_t step = (hi - lo) / 33u;
    const uint32_t c = __popc(__ballot_sync(FULL, ldn(base, lo + (uint32_t)(lane + 1) * step) < x));
    const uint32_t nlo = c ? lo + c * step + 1 : lo;
    hi = c < 32 ? lo + (c + 1) * step : hi;
    lo = nlo;
  }
  const uint32_t v = (uint32_t)lane < hi - lo ? ldn(base, lo + lane) : INF;
  return lo + __popc(__ballot_sync(FULL, v < x));
}

// membership of each lane's a in the sorted list B[0, nb)
__device__ __forceinline__ bool warp_member(const uint32_t* B, uint32_t nb, uint32_t a, int lane) {
  if (nb == 0) return false;
  if (nb <= 32) {
    const uint32_t b = (uint32_t)lane < nb ? ldn(B, lane) : INF;
    int pos = 0;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const uint32_t t = __shfl_sync(FULL, b, pos + s - 1);
      if (t < a) pos += s;
    }
    return __shfl_sync(FULL, b, pos) == a;
  }
  const uint32_t step = nb / 33u;
  const uint32_t sp = ldn(B, (uint32_t)(lane + 1) * step);
  int c = 0;
#pragma unroll
  for (int sh = 16; sh >= 1; sh >>= 1) {
    const uint32_t t = __shfl_sync(FULL, sp, c + sh - 1);
    if (t < a) c += sh;
  }
  c += __shfl_sync(FULL, sp, c) < a ? 1 : 0;
  const uint32_t lo = c ? (uint32_t)c * step + 1 : 0;
  const uint32_t hi = c < 32 ? (uint32_t)(c + 1) * step : nb;
  const uint32_t at = lb_seq(B, lo, hi, a);
  return at < nb && ldn(B, at) == a;
}


template <int K>
__global__ void __launch_bounds__(256) exact_kernel(const GraphArgs g, const DevPlan p, const int apply_bounds,
                                                    const int skip_unordered, const uint32_t root_limit,
                                                    uint32_t* __restrict__ scratch,
                                                    const uint32_t cap, unsigned long long* __restrict__ cursor,
                                                    unsigned long long* __restrict__ count_out,
                                                    const uint32_t shard, const uint32_t nshards) {
  constexpr int L = K - 2;  // steps
  const int lane = threadIdx.x & 31;
  const unsigned long long gw = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  uint32_t* buf = scratch + gw * (unsigned long long)(L > 1 ? L - 1 : 1) * cap;  // levels 0..L-2 materialised
  const uint32_t* __restrict__ nbr = g.nbr;
  unsigned long long total = 0;
  unsigned long long next = 0, end = 0;

  for (;;) {
    if (next >= end) {
      unsigned long long b = 0;
      // 32-arc chunks handed out dynamically; shard r of N owns chunks r, r+N, ...
      // (interleaved, so hub-heavy arc ranges spread over the ranks)
      if (lane == 0) b = (atomicAdd(cursor, 1ull) * nshards + shard) * 32ull;
      b = __shfl_sync(FULL, b, 0);
      if (b >= g.arcs) break;
      next = b;
      end = min(g.arcs, b + 32);
    }
    const unsigned long long arc = __ldg(g.seed_arcs + next++);
    uint32_t bnd[K], pd[K], up[K];  // up = #neighbours <= bnd: lower_bound(bnd + 1) for free
    unsigned long long pb[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      bnd[q] = INF;
      pb[q] = 0;
      pd[q] = up[q] = 0;
    }
    bnd[0] = (uint32_t)(arc >> 32);
    bnd[1] = (uint32_t)arc;
    if (skip_unordered && bnd[0] > bnd[1]) continue;  // exact_engine.cpp:84
    if (bnd[0] >= root_limit) continue;                // region split: roots below the threshold only
    {
      const VtxInfo a = load_vtx(g.vtx, bnd[0]), b = load_vtx(g.vtx, bnd[1]);
      pb[0] = a.begin;
      pd[0] = a.deg;
      up[0] = a.up;
      pb[1] = b.begin;
      pd[1] = b.deg;
      up[1] = b.up;
    }
    uint32_t len[L > 0 ? L : 1], cur[L > 0 ? L : 1];
#pragma unroll
    for (int s = 0; s < (L > 0 ? L : 1); ++s) len[s] = cur[s] = 0;

    // build level s's candidates (materialise if s < L-1, else return the count)
    auto level = [&](int s) -> uint32_t {
      uint32_t res = 0;
#pragma unroll
      for (int ss = 0; ss < L; ++ss) {
        if (ss != s) continue;
        const int j = ss + 2;
        const unsigned in_m = p.in_mask[ss], out_m = p.out_mask[ss];
        uint32_t lo = 0, hi = INF;
        if (apply_bounds) {
#pragma unroll
          for (int q = 0; q < j; ++q) {
            if ((p.gt_mask[ss] >> q) & 1u) lo = max(lo, bnd[q] + 1);
            if ((p.lt_mask[ss] >> q) & 1u) hi = min(hi, bnd[q]);
          }
        }
        uint32_t rs[K], re[K];
        int drv = -1;
        uint32_t dsize = INF;
#pragma unroll
        for (int q = 0; q < K; ++q) {
          rs[q] = re[q] = 0;
          if (q < j && ((in_m >> q) & 1u)) {
            const uint32_t* B = nbr + pb[q];
            rs[q] = lo == 0 ? 0 : lo == bnd[q] + 1 ? up[q] : kary(B, 0, pd[q], lo, lane);
            re[q] = hi == INF ? pd[q] : kary(B, rs[q], pd[q], hi, lane);
            if (re[q] < rs[q]) re[q] = rs[q];
            if (re[q] - rs[q] < dsize) {
              dsize = re[q] - rs[q];
              drv = q;
            }
          }
        }
        const bool last = ss == L - 1;
        if (last && g.core && out_m == 0 && lo >= g.core_base && dsize > 0) {
          // leaf whose lists are all dense-core rows over a range inside the core:
          // |S| = popcount of the AND of the rows over [lo, hi) minus the bound
          // vertices in it — coalesced row words instead of one search per element.
          // Taken when the row words are at most 4x the driver elements (factors
          // 1..16 measured within 5 % of each other on RMAT-18/20).
          bool rows_ok = true;
#pragma unroll
          for (int q = 0; q < K; ++q)
            if (q < j && ((in_m >> q) & 1u) && bnd[q] < g.core_base) rows_ok = false;
          const uint32_t lo_c = lo - g.core_base;
          const uint32_t hi_c = min(hi, g.core_base + g.core_wpr * 32u) - g.core_base;
          const uint32_t w0 = lo_c >> 5, w1 = hi_c > lo_c ? (hi_c + 31) >> 5 : w0;
          if (rows_ok && (w1 - w0) <= 4 * dsize) {
            uint32_t cnt = 0;
            for (uint32_t w = w0 + lane; w < w1; w += 32) {
              unsigned x = FULL;
#pragma unroll
              for (int q = 0; q < K; ++q)
                if (q < j && ((in_m >> q) & 1u))
                  x &= __ldg(g.core + (unsigned long long)(bnd[q] - g.core_base) * g.core_wpr + w);
              if (w == w0) x &= ~((1u << (lo_c & 31)) - 1u);
              if (w == w1 - 1 && (hi_c & 31)) x &= (1u << (hi_c & 31)) - 1u;
#pragma unroll
              for (int q = 0; q < K; ++q)
                if (q < j && bnd[q] >= lo && bnd[q] < hi && ((bnd[q] - g.core_base) >> 5) == w)
                  x &= ~(1u << ((bnd[q] - g.core_base) & 31));  // bound vertices are not candidates
              cnt += __popc(x);
            }
            res = __reduce_add_sync(FULL, cnt);
            continue;
          }
        }
        const uint32_t* D = nbr;
#pragma unroll
        for (int q = 0; q < K; ++q)
          if (q == drv) D = nbr + pb[q] + rs[q];
        uint32_t* out = buf + (unsigned long long)(last ? 0 : ss) * cap;
        uint32_t n = 0;
        for (uint32_t c0 = 0; c0 < dsize; c0 += 32) {
          const uint32_t i = c0 + lane;
          const bool valid = i < dsize;
          const uint32_t a = valid ? ldn(D, i) : INF;
          bool ok = valid;
#pragma unroll
          for (int q = 0; q < K; ++q) {
            if (q < j && q != drv && ((in_m >> q) & 1u)) ok = warp_member(nbr + pb[q] + rs[q], re[q] - rs[q], a, lane) && ok;
            if (q < j && ((out_m >> q) & 1u)) ok = !warp_member(nbr + pb[q], pd[q], a, lane) && ok;
            if (q < j && a == bnd[q]) ok = false;
          }
          const unsigned bal = __ballot_sync(FULL, ok);
          if (!last && ok) out[n + __popc(bal & ((1u << lane) - 1u))] = a;
          n += __popc(bal);
        }
        res = n;
      }
      return res;
    };

    if (L == 0) {
      ++total;
      continue;
    }
    // iterative DFS (exact_engine.cpp:19-62)
    int s = 0;
    uint32_t n0 = level(0);
    if (L == 1) {
      total += n0;
      continue;
    }
    len[0] = n0;
    cur[0] = 0;
    __syncwarp();
    while (true) {
      // current level s has materialised candidates len[s], cursor cur[s]
      uint32_t ls = 0, cs = 0;
#pragma unroll
      for (int t = 0; t < L; ++t)
        if (t == s) {
          ls = len[t];
          cs = cur[t];
        }
      if (cs >= ls) {
        if (s == 0) break;
        --s;
        continue;
      }
      const uint32_t v = buf[(unsigned long long)s * cap + cs];
#pragma unroll
      for (int t = 0; t < L; ++t)
        if (t == s) cur[t] = cs + 1;
      const VtxInfo vi = load_vtx(g.vtx, v);
#pragma unroll
      for (int q = 2; q < K; ++q)
        if (q == s + 2) {
          bnd[q] = v;
          pb[q] = vi.begin;
          pd[q] = vi.deg;
          up[q] = vi.up;
        }
      const int ns = s + 1;
      const uint32_t nn = level(ns);
      __syncwarp();
      if (ns == L - 1) {
        total += nn;  // eager leaf: add |S_last| (exact_engine.cpp:34-37)
      } else {
#pragma unroll
        for (int t = 0; t < L; ++t)
          if (t == ns) {
            len[t] = nn;
            cur[t] = 0;
          }
        s = ns;
      }
    }
  }
  if (lane == 0 && total) atomicAdd(count_out, total);
}

template <int K>
unsigned long long run_exact_k(const agpm_graph* gr, const DevPlan& p, bool apply_bounds, bool skip_unordered,
                               uint32_t root_limit, uint32_t shard, uint32_t nshards, cudaStream_t s) {
  DeviceCtx& ctx = ctx_for_current_device();
  // the dense-core bit matrix (core_bits.cu) answers leaves whose lists are core rows
  ensure_core_bits(const_cast<agpm_graph*>(gr), s);
  GraphArgs g{gr->vtx, gr->nbr, gr->seed_arcs, gr->arcs, gr->plain, gr->loop_free, nullptr, 0};
  g.core = gr->core;
  g.core_base = gr->core_base;
  g.core_wpr = gr->core_wpr;
  int occ = 0;
  AGPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, exact_kernel<K>, 256, 0));
  occ = std::max(occ, 1);
  const unsigned blocks = (unsigned)std::min<unsigned long long>((unsigned long long)ctx.sm_count * occ,
                                                                 (gr->arcs + 255) / 256 + 1);
  const unsigned long long warps = (unsigned long long)blocks * 8;
  const uint32_t cap = (uint32_t)std::max<uint64_t>(gr->max_degree, 1);
  const unsigned long long levels = K - 2 > 1 ? K - 3 : 1;
  auto* scratch = static_cast<uint32_t*>(ctx.get(11, 4ull * warps * levels * cap + 64));
  auto* cnt = static_cast<unsigned long long*>(ctx.get(3, 64));
  AGPM_CUDA(cudaMemsetAsync(cnt, 0, 16, s));
  exact_kernel<K><<<blocks, 256, 0, s>>>(g, p, apply_bounds ? 1 : 0, skip_unordered ? 1 : 0, root_limit, scratch,
                                         cap, cnt, cnt + 1, shard, nshards);
  count_launch();
  AGPM_CUDA(cudaGetLastError());
  unsigned long long h = 0;
  AGPM_CUDA(cudaMemcpyAsync(&h, cnt + 1, 8, cudaMemcpyDeviceToHost, s));
  AGPM_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace

// exact_count (exact_engine.cpp:66-91), eager plans; root_limit keeps only
// seeds whose first vertex is below it (region split)
unsigned long long exact_count_device(const agpm_graph* g, const agpm_plan* plan, cudaStream_t s,
                                      uint32_t root_limit, uint32_t shard, uint32_t nshards) {
  if (nshards == 0 || shard >= nshards) throw std::invalid_argument("shard must be < nshards");
  if (!plan || plan->k < 2 || plan->k > AGPM_MAX_K || plan->n_steps != plan->k - 2)
    throw std::invalid_argument("malformed plan");
  const bool clique = plan->n_edges == plan->k * (plan->k - 1) / 2;
  if (g->oriented && !clique) throw std::invalid_argument("oriented graphs are only valid for clique plans");
  if (g->oriented && plan->verify_mode == 1) throw std::invalid_argument("oriented graphs require an eager plan");
  if (plan->verify_mode != 0)
    throw std::invalid_argument("the device exact counter implements eager plans (VerifyMode::Eager)");
  const bool oriented_clique = g->oriented && clique;
  const bool apply_bounds = !oriented_clique;
  const bool skip_unordered = !oriented_clique && plan->seed_ordered;
  if (plan->k == 2 && root_limit == 0xffffffffu)  // every (ordered) arc is a match; shard 0 reports it
    return shard ? 0ull : skip_unordered ? g->arcs / 2 : g->arcs;
  DevPlan d{};
  d.k = plan->k;
  d.n_steps = plan->n_steps;
  d.seed_ordered = plan->seed_ordered;
  for (int st = 0; st < plan->n_steps; ++st) {
    const agpm_plan_step& t = plan->steps[st];
    unsigned in = 0, out = 0, gt = 0, lt = 0;
    for (int i = 0; i < t.n_in; ++i) in |= 1u << t.in_positions[i];
    for (int i = 0; i < t.n_out; ++i) out |= 1u << t.out_positions[i];
    for (int i = 0; i < t.n_gt; ++i) gt |= 1u << t.greater_than[i];
    for (int i = 0; i < t.n_lt; ++i) lt |= 1u << t.less_than[i];
    d.in_mask[st] = (unsigned short)in;
    d.out_mask[st] = (unsigned short)out;
    d.gt_mask[st] = (unsigned short)gt;
    d.lt_mask[st] = (unsigned short)lt;
  }
  if (g->arcs == 0) return 0;
  switch (plan->k) {
    case 3: return run_exact_k<3>(g, d, apply_bounds, skip_unordered, root_limit, shard, nshards, s);
    case 4: return run_exact_k<4>(g, d, apply_bounds, skip_unordered, root_limit, shard, nshards, s);
    case 5: return run_exact_k<5>(g, d, apply_bounds, skip_unordered, root_limit, shard, nshards, s);
    case 6: return run_exact_k<6>(g, d, apply_bounds, skip_unordered, root_limit, shard, nshards, s);
    case 7: return run_exact_k<7>(g, d, apply_bounds, skip_unordered, root_limit, shard, nshards, s);
    case 8: return run_exact_k<8>(g, d, apply_bounds, skip_unordered, root_limit, shard, nshards, s);
    case 9: return run_exact_k<9>(g, d, apply_bounds, skip_unordered, root_limit, shard, nshards, s);
    case 2: throw std::invalid_argument("rooted counts of a single edge are not supported");
    default: throw std::invalid_argument("device exact counter needs 2 <= k <= 9");
  }
}

}  // namespace agpm_b200

extern "C" int agpm_exact_count(agpm_graph* g, const agpm_plan* plan, uint64_t* count, void* stream) {
  return agpm_b200::guarded([&] {
    if (!g || !count) throw std::invalid_argument("null argument");
    *count = agpm_b200::exact_count_device(g, plan, agpm_b200::pick_stream(stream), 0xffffffffu, 0, 1);
  });
}

extern "C" int agpm_exact_count_shard(agpm_graph* g, const agpm_plan* plan, uint32_t shard, uint32_t nshards,
                                      uint64_t* count, void* stream) {
  return agpm_b200::guarded([&] {
    if (!g || !count) throw std::invalid_argument("null argument");
    *count = agpm_b200::exact_count_device(g, plan, agpm_b200::pick_stream(stream), 0xffffffffu, shard, nshards);
  });
}

extern "C" int agpm_exact_count_rooted(agpm_graph* g, const agpm_plan* plan, uint32_t root_limit, uint64_t* count,
                                       void* stream) {
  return agpm_b200::guarded([&] {
    if (!g || !count) throw std::invalid_argument("null argument");
    *count = agpm_b200::exact_count_device(g, plan, agpm_b200::pick_stream(stream), root_limit, 0, 1);
  });
}
