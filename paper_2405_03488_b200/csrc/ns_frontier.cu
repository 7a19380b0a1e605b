// Frontier (phase) sampler: the throughput strategy for large batches.
//
// A batch of samples advances through the plan one multi-list step at a time:
//
//   advance  (1 thread / sample)   seed draw, bound-restricted ranges of the
//            step's lists (per-thread lower_bound narrowed by hints: vtx.up,
//            the seed arc index, the previous pick's index), single-list steps
//            resolved inline by index arithmetic, driver = smallest range;
//            writes an IsectDesc + |driver| for the next multi-list step.
//   scan     (CUB)                  one exclusive scan of packed (bitmap words,
//            merge segments) per sample -> word-aligned bitmap slots + work offsets.
//   isect    (1 thread / segment)   merge-path intersection: the merge of the
//            driver D with each other list B is cut into fixed SEG-step
//            segments; a thread finds its start on the merge diagonal with one
//            binary search, then merges SEG steps, marking D elements absent
//            from B (present, for out-lists) in the sample's fail bitmap.
//            Equal-sized segments keep SIMT lanes busy however skewed the list
//            lengths are; pairs with |B| > 32|D| use per-element search instead.
//   pick     (1 thread / sample)    |S_j| = |D| - fails - bound vertices,
//            r = next_below(|S_j|), r-th surviving bit -> v_j, alpha *= |S_j|,
//            then `advance` to the next step.
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

constexpr uint32_t SEG = 64;        // merge steps per isect thread (<= 96: 128-bit mark window)
constexpr uint32_t SEG_SEARCH = 16; // driver elements per thread in search mode
constexpr uint32_t kSearchRatio = 32;  // |B| > 32 |D|: search instead of merge (set_ops.hpp:13)

// Per-sample intersection job, slots indexed by matching position (static indexing).
template <int K>
struct __align__(16) IsectDesc {
  unsigned long long drv;             // absolute index of the driver range start
  unsigned long long start[K - 1];    // other lists: in-lists restricted, out-lists whole
  uint32_t len[K - 1];
  uint32_t nseg[K - 1];               // isect work items for this list
  uint32_t dsize;
  uint32_t lists;                     // bit q: position q is an "other" list
  uint32_t outs;                      // bit q: ... and it is an out-list (difference)
  uint32_t search;                    // bit q: ... and it runs in search mode
  uint32_t drv_pos;                   // matching position owning the driver list
  uint32_t drv_rs;                    // driver range start relative to that list
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
  unsigned long long* work;     // cap + 1: (bitmap words << 32 | segments), 0 = not pending
  unsigned long long* offsets;  // cap + 1: exclusive scan of work
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
  A.work[i] = 0;
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
    // multi-list step: hand the intersection to the merge-path phase
    IsectDesc<K> d;
    d.drv = dbase;
    d.dsize = dsize;
    d.lists = d.outs = d.search = 0;
    uint32_t segs = 0;
#pragma unroll
    for (int q = 0; q < K - 1; ++q) {
      d.start[q] = 0;
      d.len[q] = 0;
      d.nseg[q] = 0;
      if (q < j && q != drv && (((in_m | out_m) >> q) & 1u)) {
        const bool is_out = (out_m >> q) & 1u;
        d.start[q] = is_out ? S.pb[q] : S.pb[q] + rs[q];
        d.len[q] = is_out ? S.pd[q] : re[q] - rs[q];
        d.lists |= 1u << q;
        if (is_out) d.outs |= 1u << q;
        if (d.len[q] / kSearchRatio > dsize) {
          d.search |= 1u << q;
          d.nseg[q] = (dsize + SEG_SEARCH - 1) / SEG_SEARCH;
        } else {
          d.nseg[q] = (dsize + d.len[q] + SEG - 1) / SEG;
        }
        segs += d.nseg[q];
      }
    }
    d.drv_pos = (uint32_t)drv;
    d.drv_rs = dbase_rel(S, drv, rs);
    reinterpret_cast<IsectDesc<K>*>(A.desc)[i] = d;
    A.work[i] = ((unsigned long long)((dsize + 31) >> 5) << 32) | segs;
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

__device__ __forceinline__ void flush_bits(uint32_t* words, uint32_t w, uint32_t bits) {
  if (bits) atomicOr(words + w, bits);
}

// One thread per work item (merge segment or search batch); a warp covers a
// contiguous run of items, so the owning sample is found by one k-ary search
// over the scanned offsets and then advanced linearly.
template <int K>
__global__ void __launch_bounds__(256) fr_isect_kernel(const FrontierArgs A, unsigned long long total) {
  const int lane = threadIdx.x & 31;
  const unsigned long long* __restrict__ off = A.offsets;
  const IsectDesc<K>* __restrict__ desc = reinterpret_cast<const IsectDesc<K>*>(A.desc);
  const uint32_t* __restrict__ nbr = A.g.nbr;
  const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
  for (unsigned long long base = ((blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5) * 32;
       base < total; base += nwarps * 32) {
    // sample of item `base`: last s with seg_off[s] <= base
    unsigned long long s;
    {
      unsigned long long lo = 0, hi = A.count;
      while (hi - lo > 32) {
        const unsigned long long step = (hi - lo) / 33;
        const unsigned long long pos = lo + (unsigned long long)(lane + 1) * step;
        const unsigned c = __popc(__ballot_sync(FULL, (off[pos] & 0xffffffffull) <= base));
        const unsigned long long nlo = c ? lo + c * step : lo;
        hi = c < 32 ? lo + (c + 1) * step : hi;
        lo = nlo;
      }
      const unsigned long long pos = lo + lane;
      const bool le = pos < hi && (off[pos] & 0xffffffffull) <= base;
      s = lo + __popc(__ballot_sync(FULL, le)) - 1;
    }
    const unsigned long long g = base + lane;
    if (g >= total) continue;
    while ((off[s + 1] & 0xffffffffull) <= g) ++s;
    const IsectDesc<K>& d = desc[s];  // fields read straight from L1, no local copy
    uint32_t l = (uint32_t)(g - (off[s] & 0xffffffffull));
    uint32_t* words = A.bitmap + (off[s] >> 32);
    const uint32_t* D = nbr + d.drv;
    const uint32_t nd = d.dsize;
#pragma unroll
    for (int q = 0; q < K - 1; ++q) {
      if (!((d.lists >> q) & 1u)) continue;
      if (l >= d.nseg[q]) {
        l -= d.nseg[q];
        continue;
      }
      const uint32_t* B = nbr + d.start[q];
      const uint32_t nb = d.len[q];
      const bool is_out = (d.outs >> q) & 1u;
      uint32_t cw = 0xffffffffu, acc = 0;
      if ((d.search >> q) & 1u) {
        const uint32_t i0 = l * SEG_SEARCH, i1 = min(nd, i0 + SEG_SEARCH);
        for (uint32_t i = i0; i < i1; ++i) {
          const uint32_t x = ldn(D, i);
          uint32_t lo = 0, hi = nb;
          while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (ldn(B, mid) < x) lo = mid + 1; else hi = mid;
          }
          const bool found = lo < nb && ldn(B, lo) == x;
          if ((i >> 5) != cw) {
            if (cw != 0xffffffffu) flush_bits(words, cw, acc);
            cw = i >> 5;
            acc = 0;
          }
          if (found == is_out) acc |= 1u << (i & 31);
        }
      } else {
        // merge-path: start of segment l on diagonal dg (D first on ties)
        const uint32_t dg = l * SEG;
        uint32_t lo = dg > nb ? dg - nb : 0, hi = min(dg, nd);
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (ldn(D, mid) <= ldn(B, dg - 1 - mid)) lo = mid + 1; else hi = mid;
        }
        uint32_t i = lo, jb = dg - lo;
        const uint32_t steps = min(SEG, nd + nb - dg);
        uint32_t x = i < nd ? ldn(D, i) : INF;
        uint32_t y = jb < nb ? ldn(B, jb) : INF;
        // branchless merge: every lane executes the same instruction stream;
        // marks go to a 128-bit window starting at i's word (SEG <= 96 bits past it)
        const uint32_t wbase = i >> 5;
        unsigned long long m0 = 0, m1 = 0;
        for (uint32_t t = 0; t < steps; ++t) {
          const bool take_d = x <= y;  // D first on ties: y = lower_bound(B, x) when D[i] is consumed
          const bool mark = take_d && ((x == y) == is_out);
          const uint32_t p = i - (wbase << 5);
          m0 |= (unsigned long long)(mark && p < 64) << (p & 63);
          m1 |= (unsigned long long)(mark && p >= 64) << (p & 63);
          i += take_d;
          jb += !take_d;
          const uint32_t k = take_d ? i : jb;
          const uint32_t lim = take_d ? nd : nb;
          const uint32_t* src = take_d ? D : B;
          const uint32_t v = k < lim ? ldn(src, k) : INF;
          x = take_d ? v : x;
          y = take_d ? y : v;
        }
        flush_bits(words, wbase, (uint32_t)m0);
        flush_bits(words, wbase + 1, (uint32_t)(m0 >> 32));
        flush_bits(words, wbase + 2, (uint32_t)m1);
        flush_bits(words, wbase + 3, (uint32_t)(m1 >> 32));
        break;
      }
      if (cw != 0xffffffffu) flush_bits(words, cw, acc);
      break;
    }
  }
}

template <int K>
__global__ void __launch_bounds__(256) fr_pick_kernel(const FrontierArgs A, int s_step) {
  const uint32_t* __restrict__ nbr = A.g.nbr;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < A.count;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    if (A.work[i] == 0) continue;
    const int j = s_step + 2;
    Sample<K> S(A.seed, A.first_id + i);
    load_state(A, i, S, j);
    const IsectDesc<K> d = reinterpret_cast<const IsectDesc<K>*>(A.desc)[i];
    const uint32_t dsize = d.dsize;
    const uint32_t* words = A.bitmap + (A.offsets[i] >> 32);
    uint32_t lo = 0, hi = INF;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      if (q < j && ((A.p.gt_mask[s_step] >> q) & 1u)) lo = max(lo, S.bnd[q] + 1);
      if (q < j && ((A.p.lt_mask[s_step] >> q) & 1u)) hi = min(hi, S.bnd[q]);
    }
    // bound vertices that survived the intersection are not candidates (walker.hpp:70-82)
    uint32_t ex[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      ex[q] = INF;
      if (q < j && S.bnd[q] >= lo && S.bnd[q] < hi) {
        const uint32_t o = lb_thread(nbr + d.drv, 0, dsize, S.bnd[q]);
        if (o < dsize && ldn(nbr, d.drv + o) == S.bnd[q] && !((words[o >> 5] >> (o & 31)) & 1u)) ex[q] = o;
      }
    }
    const uint32_t nw = (dsize + 31) >> 5;
    auto live = [&](uint32_t w) -> unsigned {  // surviving candidates in word w
      unsigned m = ~words[w];
      if (w == nw - 1 && (dsize & 31)) m &= (1u << (dsize & 31)) - 1u;
#pragma unroll
      for (int q = 0; q < K; ++q)
        if (ex[q] != INF && (ex[q] >> 5) == w) m &= ~(1u << (ex[q] & 31));
      return m;
    };
    unsigned long long cnt = 0;
    for (uint32_t w = 0; w < nw; ++w) cnt += __popc(live(w));
    if (cnt == 0) {
      finish(A, i, S, j, false);
      continue;
    }
    unsigned long long r = S.rng.next_below(cnt);
    uint32_t o = 0;
    for (uint32_t w = 0; w < nw; ++w) {
      const unsigned m = live(w);
      const unsigned pc = __popc(m);
      if (r < pc) {
        o = w * 32 + __fns(m, 0, (int)r + 1);
        break;
      }
      r -= pc;
    }
    S.alpha = __dmul_rn(S.alpha, (double)cnt);  // alpha *= |S_j| (ns_engine.cpp:39)
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
  size_t bytes = 0;
  auto carve = [&](size_t n) {
    size_t at = (bytes + 255) & ~size_t(255);
    bytes = at + n;
    return at;
  };
  const size_t o_ctr = carve(8 * cap), o_alpha = carve(8 * cap), o_bnd = carve(4ull * K * cap),
               o_hbo = carve(4ull * K * cap), o_hbl = carve(4ull * K * cap), o_work = carve(8 * (cap + 1)),
               o_off = carve(8 * (cap + 1)), o_desc = carve(sizeof(IsectDesc<K>) * cap);
  size_t scan_tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (const unsigned long long*)nullptr,
                                (unsigned long long*)nullptr, (int64_t)cap + 1, s);
  const size_t o_tmp = carve(scan_tmp + 256);
  char* slab = static_cast<char*>(ctx.get(9, bytes));
  A.ctr = reinterpret_cast<unsigned long long*>(slab + o_ctr);
  A.alpha = reinterpret_cast<double*>(slab + o_alpha);
  A.bnd = reinterpret_cast<uint32_t*>(slab + o_bnd);
  A.hbo = reinterpret_cast<uint32_t*>(slab + o_hbo);
  A.hbl = reinterpret_cast<uint32_t*>(slab + o_hbl);
  A.work = reinterpret_cast<unsigned long long*>(slab + o_work);
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
      AGPM_CUDA(cudaMemsetAsync(A.work + c, 0, 8, s));
      size_t tb = scan_tmp;
      AGPM_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, A.work, A.offsets, (int64_t)c + 1, s));
      AGPM_CUDA(cudaMemcpyAsync(h_total, A.offsets + c, 8, cudaMemcpyDeviceToHost, s));
      AGPM_CUDA(cudaStreamSynchronize(s));
      const unsigned long long words = *h_total >> 32, segs = *h_total & 0xffffffffull;
      if (words) {
        A.bitmap = static_cast<uint32_t*>(ctx.get(8, 4 * words + 64));
        AGPM_CUDA(cudaMemsetAsync(A.bitmap, 0, 4 * words, s));
        const unsigned long long warps = std::min<unsigned long long>((segs + 31) / 32, (unsigned long long)sms * 64);
        fr_isect_kernel<K><<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(A, segs);
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
