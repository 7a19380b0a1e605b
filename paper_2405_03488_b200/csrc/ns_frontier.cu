// Frontier (phase) sampler: the throughput strategy for large batches.
//
// A batch of samples advances through the plan one multi-list step at a time:
//
//   advance  (1 thread / sample)   seed draw, bound-restricted ranges of the
//            step's lists (per-thread lower_bound narrowed by hints: vtx.up,
//            the seed arc index, the previous pick's index), single-list steps
//            resolved inline by index arithmetic, driver = smallest range;
//            writes an IsectDesc + |driver| for the next multi-list step.
//   scan     (CUB)                  exclusive scan of |driver| -> element offsets.
//   isect    (1 lane / element)     every driver element of every sample is one
//            lane: load-balanced sample lookup, coalesced driver loads, one
//            branchless lower_bound per other list -> hit bit (ballot -> one
//            32-bit bitmap word per warp step). No per-sample serial work and
//            no idle lanes however skewed the list lengths are.
//   pick     (1 thread / sample)    popcount of the sample's bit range minus
//            bound vertices = |S_j|, r = next_below(|S_j|), r-th set bit ->
//            v_j, alpha *= |S_j|, then `advance` to the next step.
//
// Candidate sets and picks are exactly build_step_candidates +
// cand[next_below(|cand|)] (walker.hpp:30-83, ns_engine.cpp:27-53) with the
// sample's own CounterRng(seed, 0, id), so results are bit-identical to the
// warp/lane kernels and to the reference's draw_sample with workers = 1.
#include <cub/cub.cuh>

#include <algorithm>
#include <stdexcept>

#include "ns_common.cuh"

namespace agpm_b200 {

namespace {

constexpr uint32_t INF = 0xffffffffu;
constexpr int kMaxOther = AGPM_MAX_K - 2;

template <int K>
struct __align__(16) IsectDesc {
  unsigned long long drv;               // absolute index of the driver range start
  unsigned long long start[K - 2];      // other lists (in-lists restricted, out-lists whole)
  uint32_t len[K - 2];
  uint32_t n_other;
  uint32_t out_slots;                   // bit t set: slot t is an out-list (difference)
  uint32_t drv_pos;                     // matching position owning the driver list
  uint32_t drv_rs;                      // driver range start relative to that list
};

struct FrontierArgs {
  GraphArgs g;
  DevPlan p;
  unsigned long long seed, first_id, count;
  int step_multi[AGPM_MAX_K - 2];  // 1 if step s needs the intersection phase
  // per-sample state (SoA, stride cap)
  unsigned long long cap;
  unsigned long long* ctr;  // rng counter (key re-derived from the id)
  double* alpha;            // running scale; 0 once dead
  uint32_t* bnd;            // K * cap
  uint32_t* hbo;            // K * cap, hint: lower_bound(hbl) = hbo (relative)
  uint32_t* hbl;            // K * cap
  uint32_t* dsize;          // cap + 1 (|driver| of the pending step, 0 = not pending)
  unsigned long long* offsets;  // cap + 1
  void* desc;               // IsectDesc<K>[cap]
  uint32_t* bitmap;
  // outputs
  double* values;
  uint32_t* bindings;
};

__device__ __forceinline__ uint32_t lb_thread(const uint32_t* base, uint32_t lo, uint32_t hi, uint32_t x) {
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (ldn(base, mid) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// branchless lower_bound in base[0, n)
__device__ __forceinline__ uint32_t lb_branchless(const uint32_t* base, uint32_t n, uint32_t a) {
  if (n == 0) return 0;
  uint32_t b = 0;
  while (n > 1) {
    const uint32_t half = n >> 1;
    b = ldn(base, b + half - 1) < a ? b + half : b;
    n -= half;
  }
  return b + (ldn(base, b) < a ? 1u : 0u);
}

template <int K>
struct Sample {
  uint32_t bnd[K], hbo[K], hbl[K];
  unsigned long long pb[K];
  uint32_t pd[K], up[K];
  bool loaded[K];
  CounterRng rng;
  double alpha;
  __device__ Sample(unsigned long long seed, unsigned long long id) : rng(seed, 0, id) {}
};

template <int K>
__device__ __forceinline__ void ensure_vtx(const GraphArgs& g, Sample<K>& S, int q) {
#pragma unroll
  for (int t = 0; t < K; ++t)
    if (t == q && !S.loaded[t]) {
      const VtxInfo vi = load_vtx(g.vtx, S.bnd[t]);
      S.pb[t] = vi.begin;
      S.pd[t] = vi.deg;
      S.up[t] = vi.up;
      S.loaded[t] = true;
    }
}

template <int K>
__device__ __forceinline__ uint32_t lbq(const uint32_t* nbr, Sample<K>& S, int q, uint32_t x, bool update) {
  uint32_t r = 0;
#pragma unroll
  for (int t = 0; t < K; ++t)
    if (t == q) {
      uint32_t lo = 0, hi = S.pd[t];
      if (x >= S.bnd[t] + 1) lo = max(lo, S.up[t]); else hi = min(hi, S.up[t]);
      if (x >= S.hbl[t]) lo = max(lo, S.hbo[t]); else hi = min(hi, S.hbo[t]);
      r = x == S.hbl[t] ? S.hbo[t] : lb_thread(nbr + S.pb[t], lo, hi, x);
      if (update) {
        S.hbo[t] = r;
        S.hbl[t] = x;
      }
    }
  return r;
}

template <int K>
__device__ __forceinline__ void bind(Sample<K>& S, int q, uint32_t v) {
#pragma unroll
  for (int t = 0; t < K; ++t)
    if (t == q) {
      S.bnd[t] = v;
      S.loaded[t] = false;
      S.hbl[t] = 0;  // "no dynamic hint": lower_bound(0) = 0 always holds
      S.hbo[t] = 0;
    }
}

template <int K>
__device__ void store_state(const FrontierArgs& A, unsigned long long i, const Sample<K>& S, int nb) {
#pragma unroll
  for (int q = 0; q < K; ++q)
    if (q < nb) {
      A.bnd[q * A.cap + i] = S.bnd[q];
      A.hbo[q * A.cap + i] = S.hbo[q];
      A.hbl[q * A.cap + i] = S.hbl[q];
    }
  A.ctr[i] = S.rng.ctr;
  A.alpha[i] = S.alpha;
}

template <int K>
__device__ void load_state(const FrontierArgs& A, unsigned long long i, Sample<K>& S, int nb) {
#pragma unroll
  for (int q = 0; q < K; ++q) {
    S.loaded[q] = false;
    if (q < nb) {
      S.bnd[q] = A.bnd[q * A.cap + i];
      S.hbo[q] = A.hbo[q * A.cap + i];
      S.hbl[q] = A.hbl[q * A.cap + i];
    } else {
      S.bnd[q] = INF;
      S.hbo[q] = S.hbl[q] = 0;
    }
  }
  S.rng.ctr = A.ctr[i];
  S.alpha = A.alpha[i];
}

template <int K>
__device__ void finish(const FrontierArgs& A, unsigned long long i, const Sample<K>& S, int nb, bool hit) {
  A.values[i] = hit ? S.alpha : 0.0;
  A.dsize[i] = 0;
  if (A.bindings) {
#pragma unroll
    for (int q = 0; q < K; ++q) A.bindings[i * K + q] = q < nb ? S.bnd[q] : INF;
  }
}

template <int K>
__device__ __forceinline__ uint32_t dbase_rel(const Sample<K>&, int drv, const uint32_t (&rs)[K]) {
  uint32_t r = 0;
#pragma unroll
  for (int q = 0; q < K; ++q)
    if (q == drv) r = rs[q];
  return r;
}

// Run steps from s0 on: resolve single-list steps inline, stop at the next
// multi-list step after writing its descriptor, or finish the sample.
template <int K>
__device__ void advance(const FrontierArgs& A, unsigned long long i, Sample<K>& S, int s0) {
  const uint32_t* __restrict__ nbr = A.g.nbr;
  const DevPlan& p = A.p;
#pragma unroll
  for (int s = 0; s < K - 2; ++s) {
    if (s < s0) continue;
    const int j = s + 2;
    const unsigned in_m = p.in_mask[s], out_m = p.out_mask[s];
    const unsigned gt_m = p.gt_mask[s], lt_m = p.lt_mask[s];
    uint32_t lo = 0, hi = INF;
#pragma unroll
    for (int q = 0; q < j; ++q) {
      if ((gt_m >> q) & 1u) lo = max(lo, S.bnd[q] + 1);
      if ((lt_m >> q) & 1u) hi = min(hi, S.bnd[q]);
    }
    uint32_t rs[K], re[K];
    int drv = -1, t_in = 0;
    uint32_t dsize = INF;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      rs[q] = re[q] = 0;
      if (q < j && (((in_m | out_m) >> q) & 1u)) ensure_vtx(A.g, S, q);
      if (q < j && ((in_m >> q) & 1u)) {
        ++t_in;
        rs[q] = lo ? lbq(nbr, S, q, lo, true) : 0;
        re[q] = hi == INF ? S.pd[q] : lbq(nbr, S, q, hi, false);
        if (re[q] < rs[q]) re[q] = rs[q];
        if (re[q] - rs[q] < dsize) {
          dsize = re[q] - rs[q];
          drv = q;
        }
      }
    }
    unsigned long long dbase = 0;
#pragma unroll
    for (int q = 0; q < K; ++q)
      if (q == drv) dbase = S.pb[q] + rs[q];
    if (dsize == 0) {
      finish(A, i, S, j, false);
      return;
    }
    if (!A.step_multi[s]) {
      // single list: |S| = |range| - bound vertices inside it, pick by index
      uint32_t ex[K];
      uint32_t nex = 0;
#pragma unroll
      for (int q = 0; q < K; ++q) {
        ex[q] = INF;
        if (q < j && S.bnd[q] >= lo && S.bnd[q] < hi) {
          const uint32_t o = lb_thread(nbr + dbase, 0, dsize, S.bnd[q]);
          if (o < dsize && ldn(nbr, dbase + o) == S.bnd[q]) {
            ex[q] = o;
            ++nex;
          }
        }
      }
      const uint32_t cnt = dsize - nex;
      if (cnt == 0) {
        finish(A, i, S, j, false);
        return;
      }
      const uint32_t r = (uint32_t)S.rng.next_below(cnt);
      uint32_t o = r;
      for (int it = 0; it < K; ++it) {
        uint32_t c = 0;
#pragma unroll
        for (int q = 0; q < K; ++q) c += ex[q] <= o ? 1u : 0u;
        if (r + c == o) break;
        o = r + c;
      }
      S.alpha = __dmul_rn(S.alpha, (double)cnt);
      const uint32_t pick = ldn(nbr, dbase + o);
#pragma unroll
      for (int q = 0; q < j; ++q)
        if (q == drv) {
          S.hbo[q] = rs[q] + o + 1;
          S.hbl[q] = pick + 1;
        }
      bind(S, j, pick);
      continue;
    }
    // multi-list step: hand the intersection to the element-parallel phase
    IsectDesc<K> d;
    d.drv = dbase;
    uint32_t t = 0, outs = 0;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      if (q < j && q != drv && (((in_m | out_m) >> q) & 1u) && t < K - 2) {
        const bool is_out = (out_m >> q) & 1u;
        d.start[t] = is_out ? S.pb[q] : S.pb[q] + rs[q];
        d.len[t] = is_out ? S.pd[q] : re[q] - rs[q];
        if (is_out) outs |= 1u << t;
        ++t;
      }
    }
#pragma unroll
    for (int u = 0; u < K - 2; ++u)
      if (u >= (int)t) {
        d.start[u] = 0;
        d.len[u] = 0;
      }
    d.n_other = t;
    d.out_slots = outs;
    d.drv_pos = (uint32_t)drv;
    d.drv_rs = dbase_rel(S, drv, rs);
    reinterpret_cast<IsectDesc<K>*>(A.desc)[i] = d;
    A.dsize[i] = dsize;
    store_state(A, i, S, j);
    return;
  }
  finish(A, i, S, K, true);
}

template <int K>
__global__ void __launch_bounds__(256) fr_seed_kernel(const FrontierArgs A) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < A.count;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    Sample<K> S(A.seed, A.first_id + i);
#pragma unroll
    for (int q = 0; q < K; ++q) {
      S.bnd[q] = INF;
      S.hbo[q] = S.hbl[q] = 0;
      S.loaded[q] = false;
      S.pb[q] = 0;
      S.pd[q] = S.up[q] = 0;
    }
    S.alpha = A.p.alpha0;
    const unsigned long long r0 = S.rng.next_below(A.g.arcs);
    const unsigned long long arc = __ldg(A.g.seed_arcs + r0);
    uint32_t u = (uint32_t)(arc >> 32), v = (uint32_t)arc;
    const bool swapped = A.p.seed_ordered && u > v;
    if (swapped) {
      const uint32_t t = u;
      u = v;
      v = t;
    }
    bind(S, 0, u);
    bind(S, 1, v);
    ensure_vtx(A.g, S, 0);
    ensure_vtx(A.g, S, 1);
    if (A.g.plain) {  // arc r0 is nbr[r0] in its source's list
      if (!swapped) {
        S.hbo[0] = (uint32_t)(r0 - S.pb[0]) + 1;
        S.hbl[0] = v + 1;
      } else {
        S.hbo[1] = (uint32_t)(r0 - S.pb[1]) + 1;
        S.hbl[1] = u + 1;
      }
    }
    advance<K>(A, i, S, 0);
  }
}

// One lane per driver element; warps walk contiguous runs of bitmap words.
template <int K>
__global__ void __launch_bounds__(256) fr_isect_kernel(const FrontierArgs A, unsigned long long total) {
  const int lane = threadIdx.x & 31;
  const unsigned long long words = (total + 31) >> 5;
  const unsigned long long warp = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
  const unsigned long long per = (words + nwarps - 1) / nwarps;
  const unsigned long long w0 = warp * per, w1 = min(words, w0 + per);
  if (w0 >= w1) return;
  const unsigned long long* __restrict__ off = A.offsets;
  const IsectDesc<K>* __restrict__ desc = reinterpret_cast<const IsectDesc<K>*>(A.desc);
  const uint32_t* __restrict__ nbr = A.g.nbr;
  // sample holding element 32*w0: last s with off[s] <= 32*w0 (k-ary over the offsets)
  unsigned long long s_cur;
  {
    const unsigned long long e0 = w0 * 32;
    unsigned long long lo = 0, hi = A.count;  // answer in [lo, hi)
    while (hi - lo > 32) {
      const unsigned long long step = (hi - lo) / 33;
      const unsigned long long pos = lo + (unsigned long long)(lane + 1) * step;
      const unsigned bal = __ballot_sync(FULL, off[pos] <= e0);
      const unsigned c = __popc(bal);
      const unsigned long long nlo = c ? lo + c * step : lo;
      hi = c < 32 ? lo + (c + 1) * step : hi;
      lo = nlo;
    }
    const unsigned long long pos = lo + lane;
    const bool le = pos < hi && off[pos] <= e0;
    s_cur = lo + __popc(__ballot_sync(FULL, le)) - 1;
  }
  for (unsigned long long w = w0; w < w1; ++w) {
    const unsigned long long e = w * 32 + lane;
    const bool valid = e < total;
    unsigned long long s = s_cur;
    if (valid)
      while (off[s + 1] <= e) ++s;
    bool ok = false;
    if (valid) {
      const IsectDesc<K> d = desc[s];
      const uint32_t a = ldn(nbr, d.drv + (e - off[s]));
      ok = true;
#pragma unroll
      for (int t = 0; t < K - 2; ++t) {
        if ((uint32_t)t < d.n_other) {
          const uint32_t* B = nbr + d.start[t];
          const uint32_t o = lb_branchless(B, d.len[t], a);
          const bool found = o < d.len[t] && ldn(B, o) == a;
          ok = ok && (((d.out_slots >> t) & 1u) ? !found : found);
        }
      }
    }
    const unsigned bal = __ballot_sync(FULL, ok);
    if (lane == 0) A.bitmap[w] = bal;
    s_cur = __shfl_sync(FULL, s, 31);  // lane 31 holds the largest sample of this word
  }
}

template <int K>
__global__ void __launch_bounds__(256) fr_pick_kernel(const FrontierArgs A, int s_step) {
  const uint32_t* __restrict__ nbr = A.g.nbr;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < A.count;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t dsize = A.dsize[i];
    if (dsize == 0) continue;
    const int j = s_step + 2;
    Sample<K> S(A.seed, A.first_id + i);
    load_state(A, i, S, j);
    const IsectDesc<K> d = reinterpret_cast<const IsectDesc<K>*>(A.desc)[i];
    const unsigned long long off = A.offsets[i];
    // order bounds of this step (bound vertices outside them cannot be candidates)
    uint32_t lo = 0, hi = INF;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      if (q < j && ((A.p.gt_mask[s_step] >> q) & 1u)) lo = max(lo, S.bnd[q] + 1);
      if (q < j && ((A.p.lt_mask[s_step] >> q) & 1u)) hi = min(hi, S.bnd[q]);
    }
    // bound vertices that survived the intersection are not candidates
    uint32_t ex[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      ex[q] = INF;
      if (q < j && S.bnd[q] >= lo && S.bnd[q] < hi) {
        const uint32_t o = lb_thread(nbr + d.drv, 0, dsize, S.bnd[q]);
        if (o < dsize && ldn(nbr, d.drv + o) == S.bnd[q]) {
          const unsigned long long bit = off + o;
          if ((A.bitmap[bit >> 5] >> (bit & 31)) & 1u) ex[q] = o;
        }
      }
    }
    auto word_at = [&](unsigned long long w) -> unsigned {
      unsigned m = A.bitmap[w];
      const unsigned long long b0 = w * 32;
      if (b0 < off) m &= ~0u << (off - b0);
      const unsigned long long end = off + dsize;
      if (b0 + 32 > end) m &= end - b0 >= 32 ? ~0u : ((1u << (end - b0)) - 1u);
#pragma unroll
      for (int q = 0; q < K; ++q)
        if (ex[q] != INF) {
          const unsigned long long bit = off + ex[q];
          if ((bit >> 5) == w) m &= ~(1u << (bit & 31));
        }
      return m;
    };
    const unsigned long long wa = off >> 5, wb = (off + dsize - 1) >> 5;
    unsigned long long cnt = 0;
    for (unsigned long long w = wa; w <= wb; ++w) cnt += __popc(word_at(w));
    if (cnt == 0) {
      finish(A, i, S, j, false);
      continue;
    }
    unsigned long long r = S.rng.next_below(cnt);
    uint32_t o = 0;
    for (unsigned long long w = wa; w <= wb; ++w) {
      const unsigned m = word_at(w);
      const unsigned pc = __popc(m);
      if (r < pc) {
        o = (uint32_t)(w * 32 + __fns(m, 0, (int)r + 1) - off);
        break;
      }
      r -= pc;
    }
    S.alpha = __dmul_rn(S.alpha, (double)cnt);
    const uint32_t pick = ldn(nbr, d.drv + o);
    // the pick sits at drv_rs + o in the driver's list: lower_bound(pick+1) = drv_rs + o + 1
#pragma unroll
    for (int q = 0; q < K; ++q)
      if ((uint32_t)q == d.drv_pos) {
        S.hbo[q] = d.drv_rs + o + 1;
        S.hbl[q] = pick + 1;
      }
    bind(S, j, pick);
    advance<K>(A, i, S, s_step + 1);
  }
}

template <int K>
void run_frontier_k(const SampleLaunch& L, cudaStream_t s) {
  DeviceCtx& ctx = ctx_for_current_device();
  FrontierArgs A{};
  A.g = L.g;
  A.p = L.p;
  A.seed = L.seed;
  for (int st = 0; st < K - 2; ++st) {
    const unsigned in_m = L.p.in_mask[st], out_m = L.p.out_mask[st];
    A.step_multi[st] = !(__builtin_popcount(in_m) == 1 && out_m == 0);
  }
  const unsigned long long cap = std::min<unsigned long long>(L.count, 1ull << 22);
  A.cap = cap;
  // state slab in scratch slot 6
  size_t bytes = 0;
  auto carve = [&](size_t n) {
    size_t at = (bytes + 255) & ~size_t(255);
    bytes = at + n;
    return at;
  };
  const size_t o_ctr = carve(8 * cap), o_alpha = carve(8 * cap), o_bnd = carve(4ull * K * cap),
               o_hbo = carve(4ull * K * cap), o_hbl = carve(4ull * K * cap), o_dsize = carve(4 * (cap + 1)),
               o_off = carve(8 * (cap + 1)), o_desc = carve(sizeof(IsectDesc<K>) * cap);
  size_t scan_tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (const uint32_t*)nullptr, (unsigned long long*)nullptr,
                                (int64_t)cap + 1, s);
  const size_t o_tmp = carve(scan_tmp + 256);
  char* slab = static_cast<char*>(ctx.get(9, bytes));
  A.ctr = reinterpret_cast<unsigned long long*>(slab + o_ctr);
  A.alpha = reinterpret_cast<double*>(slab + o_alpha);
  A.bnd = reinterpret_cast<uint32_t*>(slab + o_bnd);
  A.hbo = reinterpret_cast<uint32_t*>(slab + o_hbo);
  A.hbl = reinterpret_cast<uint32_t*>(slab + o_hbl);
  A.dsize = reinterpret_cast<uint32_t*>(slab + o_dsize);
  A.offsets = reinterpret_cast<unsigned long long*>(slab + o_off);
  A.desc = slab + o_desc;
  void* tmp = slab + o_tmp;
  auto* h_total = static_cast<unsigned long long*>(ctx.get_pinned(2, 64));

  const int sms = ctx.sm_count;
  for (unsigned long long done = 0; done < L.count; done += cap) {
    const unsigned long long c = std::min(cap, L.count - done);
    A.count = c;
    A.first_id = L.first_id + done;
    A.values = L.values + done;
    A.bindings = L.bindings ? L.bindings + done * K : nullptr;
    const unsigned blocks = (unsigned)std::min<unsigned long long>((c + 255) / 256, (unsigned long long)sms * 16);
    fr_seed_kernel<K><<<blocks, 256, 0, s>>>(A);
    count_launch();
    AGPM_CUDA(cudaGetLastError());
    for (int st = 0; st < K - 2; ++st) {
      if (!A.step_multi[st]) continue;
      AGPM_CUDA(cudaMemsetAsync(A.dsize + c, 0, 4, s));
      size_t tb = scan_tmp;
      AGPM_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, A.dsize, A.offsets, (int64_t)c + 1, s));
      AGPM_CUDA(cudaMemcpyAsync(h_total, A.offsets + c, 8, cudaMemcpyDeviceToHost, s));
      AGPM_CUDA(cudaStreamSynchronize(s));
      const unsigned long long total = *h_total;
      if (total) {
        const unsigned long long words = (total + 31) >> 5;
        A.bitmap = static_cast<uint32_t*>(ctx.get(8, 4 * words + 64));
        const unsigned long long warps = std::min<unsigned long long>((words + 3) / 4, (unsigned long long)sms * 64);
        fr_isect_kernel<K><<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(A, total);
        count_launch();
        AGPM_CUDA(cudaGetLastError());
      }
      fr_pick_kernel<K><<<blocks, 256, 0, s>>>(A, st);
      count_launch();
      AGPM_CUDA(cudaGetLastError());
    }
  }
}

}  // namespace

void launch_ns_frontier(const SampleLaunch& L, cudaStream_t s) {
  if (L.bytes_out) throw std::invalid_argument("B_min accounting runs on the warp sampler");
#define AGPM_K(KK)          \
  case KK:                  \
    run_frontier_k<KK>(L, s); \
    break;
  switch (L.p.k) {
    AGPM_K(3)
    AGPM_K(4)
    AGPM_K(5)
    AGPM_K(6)
    AGPM_K(7)
    AGPM_K(8)
    AGPM_K(9)
    default:
      throw std::invalid_argument("device sampler needs 3 <= k <= 9");
  }
#undef AGPM_K
}

}  // namespace agpm_b200
