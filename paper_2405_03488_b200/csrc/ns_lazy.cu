// Lazy-verify neighbour sampling (NS-base, VerifyMode::Lazy): ONE warp per sample.
//
// The paper's baseline sampler. Step j's candidate set is the UNION of the
// adjacency lists of every bound vertex, minus the bound vertices, with no
// id-order bounds (walker.hpp:56-62 with apply_bounds ignored for Lazy); the
// pick is S[next_below(|S|)] in ascending order and only its tree-parent edge
// is checked on the spot (ns_engine.cpp:41-46). After the last step the
// closure edges, the terminal order constraints and — for vertex-induced
// patterns — the absent edges are verified (walker.hpp:88-107).
//
// The union is streamed, never materialised: per iteration the warp loads the
// next 32 elements of every list; F = the smallest "last loaded element" over
// lists that still have unloaded elements, so every union element <= F sits
// in a loaded chunk. An element is emitted by the first list (in position
// order) that holds it — membership in earlier chunks is a shuffle search —
// and each list advances past its elements <= F. Pass 1 counts |S|; pass 2
// re-streams up to the chunk holding the r-th element and finds it by rank
// (rank = sum over lists of emitted elements below it). Bit-identical to the
// reference's draw_sample for lazy plans (values, hits, bindings).
#include <algorithm>
#include <stdexcept>

#include "ns_common.cuh"

namespace agpm_b200 {
namespace {

constexpr int kLazyBatch = 4;

template <int K>
struct LazyState {
  uint32_t bnd[K];
  unsigned long long pb[K];
  uint32_t pd[K];
};

// Streams the union of the lists of positions [0, j). With target == ~0 it
// returns |S|; otherwise it stops at the target-th element (0-based) of S and
// writes it to *pick.
template <int K>
__device__ __forceinline__ unsigned long long union_scan(const LazyState<K>& st, const uint32_t* __restrict__ nbr,
                                                         int j, unsigned long long target, int lane,
                                                         uint32_t* pick) {
  uint32_t cur[K];
#pragma unroll
  for (int q = 0; q < K; ++q) cur[q] = 0;
  unsigned long long before = 0;
  for (;;) {
    uint32_t val[K];
    uint32_t F = kNoVertex;
    bool any = false;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      val[q] = kNoVertex;
      if (q < j) {
        const uint32_t rem = st.pd[q] - cur[q];
        if ((uint32_t)lane < rem) val[q] = ldn(nbr, st.pb[q] + cur[q] + lane);
        if (rem > 32) F = min(F, __shfl_sync(FULL, val[q], 31));
        any = any || rem > 0;
      }
    }
    if (!any) break;
    unsigned em[K];
    unsigned long long cnt = 0;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      em[q] = 0;
      if (q < j) {
        const uint32_t x = val[q];
        bool ok = x != kNoVertex && x <= F;
#pragma unroll
        for (int t = 0; t < K; ++t) {
          if (t < q) {
            const bool dup = chunk_contains(val[t], x);  // every lane shuffles: no short-circuit
            ok = ok && !dup;
          }
          if (t < j) ok = ok && x != st.bnd[t];
        }
        em[q] = __ballot_sync(FULL, ok);
        cnt += __popc(em[q]);
      }
    }
    if (target != ~0ull && target < before + cnt) {
      const uint32_t rr = (uint32_t)(target - before);
#pragma unroll
      for (int q = 0; q < K; ++q) {
        if (q < j) {
          const uint32_t x = val[q];
          uint32_t rank = 0;
#pragma unroll
          for (int t = 0; t < K; ++t) {
            if (t < j) {
              const uint32_t p = chunk_rank(val[t], x);
              rank += __popc(em[t] & (p >= 32 ? FULL : ((1u << p) - 1u)));
            }
          }
          const unsigned who = __ballot_sync(FULL, ((em[q] >> lane) & 1u) && rank == rr);
          if (who) {
            *pick = __shfl_sync(FULL, x, __ffs(who) - 1);
            return target;
          }
        }
      }
    }
    before += cnt;
#pragma unroll
    for (int q = 0; q < K; ++q)
      if (q < j) cur[q] += __popc(__ballot_sync(FULL, val[q] != kNoVertex && val[q] <= F));
  }
  return before;
}

// has_arc(u, v): v in u's list (k-ary search, warp-uniform)
template <int K>
__device__ __forceinline__ bool has_arc_w(const GraphArgs& g, uint32_t u, uint32_t v, int lane) {
  const VtxInfo vi = load_vtx(g.vtx, u);
  bool f = false;
  kary_lb(g.nbr + vi.begin, 0, vi.deg, v, lane, &f);
  return f;
}

template <int K>
__global__ void __launch_bounds__(256) ns_lazy_kernel(const SampleLaunch L) {
  const int lane = threadIdx.x & 31;
  const DevPlan& p = L.p;
  unsigned long long next = 0, end = 0;
  for (;;) {
    if (next >= end) {
      unsigned long long b = 0;
      if (lane == 0) b = atomicAdd(L.cursor, (unsigned long long)kLazyBatch);
      b = __shfl_sync(FULL, b, 0);
      if (b >= L.count) break;
      next = b;
      end = min(L.count, b + kLazyBatch);
    }
    const unsigned long long idx = next++;
    CounterRng rng(L.seed, 0, L.first_id + idx);
    LazyState<K> st;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      st.bnd[q] = kNoVertex;
      st.pb[q] = 0;
      st.pd[q] = 0;
    }
    auto bind = [&](int q, uint32_t v) {
      const VtxInfo vi = load_vtx(L.g.vtx, v);
#pragma unroll
      for (int t = 0; t < K; ++t)
        if (t == q) {
          st.bnd[t] = v;
          st.pb[t] = vi.begin;
          st.pd[t] = vi.deg;
        }
    };
    // seed (ns_engine.cpp:29-33)
    {
      const unsigned long long r0 = rng.next_below(L.g.arcs);
      const unsigned long long arc = __ldg(L.g.seed_arcs + r0);
      uint32_t u = (uint32_t)(arc >> 32), v = (uint32_t)arc;
      if (p.seed_ordered && u > v) {
        const uint32_t t = u;
        u = v;
        v = t;
      }
      bind(0, u);
      bind(1, v);
    }
    double alpha = p.alpha0;
    bool alive = true;
    int nbound = 2;
#pragma unroll
    for (int s = 0; s < K - 2; ++s) {
      if (!alive) break;
      const int j = s + 2;
      uint32_t pick = kNoVertex;
      const unsigned long long cnt = union_scan<K>(st, L.g.nbr, j, ~0ull, lane, &pick);
      if (cnt == 0) {
        alive = false;
        break;
      }
      const unsigned long long r = rng.next_below(cnt);
      union_scan<K>(st, L.g.nbr, j, r, lane, &pick);
      alpha = __dmul_rn(alpha, (double)cnt);  // ns_engine.cpp:39
      bind(j, pick);
      nbound = j + 1;
      uint32_t parent = 0;
#pragma unroll
      for (int q = 0; q < K; ++q)
        if (q == p.tree_parent[s]) parent = st.bnd[q];
      if (!has_arc_w<K>(L.g, parent, pick, lane)) alive = false;  // ns_engine.cpp:41-46
    }
    if (alive) {  // walker.hpp:88-107
      auto at = [&](int q) {
        uint32_t v = 0;
#pragma unroll
        for (int t = 0; t < K; ++t)
          if (t == q) v = st.bnd[t];
        return v;
      };
      for (int i = 0; i < p.n_closure && alive; ++i)
        alive = has_arc_w<K>(L.g, at(p.closure[i][0]), at(p.closure[i][1]), lane);
      for (int i = 0; i < p.n_terminal && alive; ++i) alive = at(p.terminal[i][0]) < at(p.terminal[i][1]);
      for (int i = 0; i < p.n_nonadj && alive; ++i)
        alive = !has_arc_w<K>(L.g, at(p.nonadj[i][0]), at(p.nonadj[i][1]), lane);
    }
    if (lane == 0) L.values[idx] = alive ? alpha : 0.0;
    if (L.bindings) {
#pragma unroll
      for (int q = 0; q < K; ++q)
        if (lane == q) L.bindings[idx * K + q] = q < nbound ? st.bnd[q] : kNoVertex;
    }
  }
}

template <int K>
void launch_lazy_k(const SampleLaunch& L, cudaStream_t s) {
  DeviceCtx& ctx = ctx_for_current_device();
  static int occ = -1;
  if (occ < 0) {
    int o = 0;
    AGPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, ns_lazy_kernel<K>, 256, 0));
    occ = o > 0 ? o : 1;
  }
  const uint64_t warps_needed = (L.count + kLazyBatch - 1) / kLazyBatch;
  uint64_t blocks = std::min<uint64_t>((uint64_t)ctx.sm_count * occ, (warps_needed + 7) / 8);
  if (blocks == 0) blocks = 1;
  ns_lazy_kernel<K><<<(unsigned)blocks, 256, 0, s>>>(L);
  count_launch();
  AGPM_CUDA(cudaGetLastError());
}

}  // namespace

void launch_ns_lazy(const SampleLaunch& L, cudaStream_t s) {
  switch (L.p.k) {
    case 3: launch_lazy_k<3>(L, s); break;
    case 4: launch_lazy_k<4>(L, s); break;
    case 5: launch_lazy_k<5>(L, s); break;
    case 6: launch_lazy_k<6>(L, s); break;
    case 7: launch_lazy_k<7>(L, s); break;
    case 8: launch_lazy_k<8>(L, s); break;
    case 9: launch_lazy_k<9>(L, s); break;
    default: throw std::invalid_argument("device sampler needs 3 <= k <= 9");
  }
}

}  // namespace agpm_b200
