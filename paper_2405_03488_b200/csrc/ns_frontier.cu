// Frontier (phase) sampler: the throughput strategy for large batches.
//
// A batch of samples advances through the plan one multi-list step at a time:
//
//   advance  (1 thread / sample)   seed draw; bound-restricted ranges of the
//            step's lists (per-thread lower_bound narrowed by hints: vtx.up,
//            the seed arc index, the previous pick's index); single-list steps
//            resolved inline by index arithmetic; driver = smallest range;
//            writes an IsectDesc and the sample's bitmap word count.
//   scan     (CUB)                  word offsets: every sample's hit bitmap
//            starts on a 32-bit word boundary.
//   isect    (1 warp / bitmap word) a word = 32 driver elements of ONE sample.
//            Every "a in list q" test is one probe of the device edge table
//            (edge_hash.cuh: one 32-B bucket per lookup), since the driver
//            already sits inside the step's [lo, hi). Without a table the warp
//            loads 32 splitters of list q, finds each lane's bucket with a
//            5-step shuffle search and finishes with a short per-lane search.
//            One ballot -> the fail word. No atomics, no memset.
//   pick     (1 thread / sample)    |S_j| = |D| - fails - bound vertices,
//            r = next_below(|S_j|), r-th surviving bit -> v_j, alpha *= |S_j|.
//            Nested reuse: when step j+1's lists contain step j's (cliques),
//            S_{j+1} = {x in S_j : x in [lo', hi'), x != v_j} ∩ (new lists) —
//            the survivors are compacted (warp-aggregated allocation) and become
//            the next driver, so step j+1 intersects a handful of elements
//            with ONE new list instead of re-intersecting all of them.
//
// Candidate sets and picks are exactly build_step_candidates +
// cand[next_below(|cand|)] (walker.hpp:30-83, ns_engine.cpp:27-53) with the
// sample's own CounterRng(seed, 0, id): the set S_j does not depend on how it
// is computed, so results are bit-identical to the warp/lane kernels and to the
// reference's draw_sample with workers = 1.
#include <cub/cub.cuh>

#include <algorithm>
#include <stdexcept>

#include "edge_hash.cuh"
#include "ns_common.cuh"

namespace agpm_b200 {

namespace {

constexpr uint32_t INF = 0xffffffffu;
constexpr unsigned long long kFrontierCap = 1ull << 24;  // samples per pass
constexpr uint32_t NO_DRV = 0xffffffffu;

// Per-sample intersection job; other-list slots are indexed by matching position.
template <int K>
struct __align__(16) IsectDesc {
  const uint32_t* drv;                // driver list (adjacency range or compacted survivors)
  unsigned long long start[K - 1];    // other lists: in-lists restricted, out-lists whole
  uint32_t len[K - 1];
  uint32_t owner[K - 1];              // bound vertex whose adjacency list slot q is
  uint32_t dsize;
  uint32_t lists;                     // bit q: position q is an other list
  uint32_t outs;                      // bit q: ... and an out-list (difference)
  uint32_t drv_pos;                   // position owning the driver list, NO_DRV for survivors
  uint32_t drv_rs;                    // driver range start relative to that list
  uint32_t core;                      // bit q: list q's owner is a core vertex; bit 31: driver >= core base
};

struct FrontierArgs {
  GraphArgs g;
  DevPlan p;
  unsigned long long seed, first_id, count;
  int step_multi[AGPM_MAX_K - 2];  // step s needs the intersection phase
  int step_reuse[AGPM_MAX_K - 2];  // step s reuses step s-1's survivors as its driver
  // per-sample state (SoA, stride cap)
  unsigned long long cap;
  unsigned long long* ctr;      // rng counter (key re-derived from the id)
  double* alpha;                // running scale
  uint32_t* bnd;                // K * cap
  uint32_t* hbo;                // K * cap, hint: lower_bound(hbl) = hbo (relative)
  uint32_t* hbl;                // K * cap
  unsigned long long* work;     // cap + 1: bitmap words of the pending step, 0 = not pending
  unsigned long long* offsets;  // cap + 1: exclusive scan of work
  void* desc;                   // IsectDesc<K>[cap]
  uint32_t* bitmap;             // fail bits
  uint32_t* survivors[2];       // compacted survivor lists (double-buffered by step parity)
  unsigned long long* surv_cursor;  // [2] allocation cursors
  unsigned long long surv_cap;
  // outputs
  double* values;
  uint32_t* bindings;
};

__device__ __forceinline__ uint32_t lb_thread(const uint32_t* base, uint32_t lo, uint32_t hi, uint32_t x) {
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (ldo(base, mid) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

template <int K>
struct Sample {
  uint32_t bnd[K], hbo[K], hbl[K];
  unsigned long long pb[K];
  uint32_t pd[K], up[K];
  bool loaded[K];
  CounterRng rng;
  double alpha;
  __device__ Sample(unsigned long long seed, unsigned long long id) : rng(seed, 0, id) {
#pragma unroll
    for (int q = 0; q < K; ++q) {
      bnd[q] = INF;
      hbo[q] = hbl[q] = 0;
      loaded[q] = false;
      pb[q] = 0;
      pd[q] = up[q] = 0;
    }
    alpha = 0.0;
  }
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
  for (int q = 0; q < K; ++q)
    if (q < nb) {
      S.bnd[q] = A.bnd[q * A.cap + i];
      S.hbo[q] = A.hbo[q * A.cap + i];
      S.hbl[q] = A.hbl[q * A.cap + i];
    }
  S.rng.ctr = A.ctr[i];
  S.alpha = A.alpha[i];
}

template <int K>
__device__ void finish(const FrontierArgs& A, unsigned long long i, const Sample<K>& S, int nb, bool hit) {
  A.values[i] = hit ? S.alpha : 0.0;
  if (A.work) A.work[i] = 0;
  if (A.bindings) {
#pragma unroll
    for (int q = 0; q < K; ++q) A.bindings[i * K + q] = q < nb ? S.bnd[q] : INF;
  }
}

// order bounds of step s from the current bindings (walker.hpp:64-69)
template <int K>
__device__ __forceinline__ void step_bounds(const DevPlan& p, int s, const Sample<K>& S, uint32_t& lo, uint32_t& hi) {
  lo = 0;
  hi = INF;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    if (q < s + 2 && ((p.gt_mask[s] >> q) & 1u)) lo = max(lo, S.bnd[q] + 1);
    if (q < s + 2 && ((p.lt_mask[s] >> q) & 1u)) hi = min(hi, S.bnd[q]);
  }
}

// Run steps from s0 on: resolve single-list steps inline, stop at the next
// multi-list step after writing its descriptor, or finish the sample. With
// `surv` set, step s0 uses those survivors of step s0-1 as its driver and only
// the lists step s0-1 did not have.
// Returns the step whose descriptor was written (pending intersection), or -1
// once the sample is finished. With `local` set (fused kernel) the descriptor
// goes there and nothing is written to the SoA state.
template <int K>
__device__ int advance(const FrontierArgs& A, unsigned long long i, Sample<K>& S, int s0, const uint32_t* surv,
                       uint32_t surv_len, IsectDesc<K>* local = nullptr) {
  const uint32_t* __restrict__ nbr = A.g.nbr;
  const DevPlan& p = A.p;
#pragma unroll
  for (int s = 0; s < K - 2; ++s) {
    if (s < s0) continue;
    const int j = s + 2;
    const bool reuse = s == s0 && surv != nullptr;
    const unsigned prev_in = reuse && s > 0 ? p.in_mask[s - 1] : 0u;
    const unsigned prev_out = reuse && s > 0 ? p.out_mask[s - 1] : 0u;
    const unsigned in_m = p.in_mask[s] & ~prev_in, out_m = p.out_mask[s] & ~prev_out;
    uint32_t lo, hi;
    step_bounds(p, s, S, lo, hi);
    // Ranges [rs, re) of the in-lists inside [lo, hi). First a SUPERSET range
    // from the hints alone (no memory traffic): up = lower_bound(bnd + 1) and
    // hbo = lower_bound(hbl) bracket lower_bound(lo) / lower_bound(hi). Only the
    // driver needs its exact range (it is enumerated); other lists are probed
    // for membership of elements already inside [lo, hi), for which a superset
    // range answers the same. Exact ranges are computed smallest-superset first
    // until the smallest candidate is exact, so the driver is still the
    // smallest exact range.
    uint32_t rs[K], re[K];
    bool exact[K];
    int drv = -1, t_in = 0;
    uint32_t dsize = INF;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      rs[q] = re[q] = 0;
      exact[q] = false;
      if (q < j && (((in_m | out_m) >> q) & 1u)) ensure_vtx(A.g, S, q);
      if (q < j && ((in_m >> q) & 1u)) {
        ++t_in;
        uint32_t L = 0, U = S.pd[q];
        bool ex_lo = lo == 0, ex_hi = hi == INF;
        if (lo) {
          if (lo >= S.bnd[q] + 1) L = max(L, S.up[q]);
          if (lo >= S.hbl[q]) L = max(L, S.hbo[q]);
          ex_lo = lo == S.bnd[q] + 1 || lo == S.hbl[q];
        }
        if (hi != INF) {
          if (hi <= S.bnd[q] + 1) U = min(U, S.up[q]);
          if (hi <= S.hbl[q]) U = min(U, S.hbo[q]);
          ex_hi = hi == S.bnd[q] + 1 || hi == S.hbl[q];
        }
        rs[q] = L;
        re[q] = max(U, L);
        exact[q] = ex_lo && ex_hi;
      }
    }
    if (!reuse) {
#pragma unroll
      for (int it = 0; it < K; ++it) {
        int b = -1;
        uint32_t bs = INF;
        bool bex = false;
#pragma unroll
        for (int q = 0; q < K; ++q)
          if (q < j && ((in_m >> q) & 1u) && re[q] - rs[q] < bs) {
            bs = re[q] - rs[q];
            b = q;
            bex = exact[q];
          }
        if (b < 0) break;
        if (bex) {
          drv = b;
          dsize = bs;
          break;
        }
#pragma unroll
        for (int q = 0; q < K; ++q)
          if (q == b) {
            rs[q] = lo ? lbq(nbr, S, q, lo, true) : 0;
            re[q] = hi == INF ? S.pd[q] : lbq(nbr, S, q, hi, false);
            if (re[q] < rs[q]) re[q] = rs[q];
            exact[q] = true;
          }
      }
    }
    const uint32_t* dptr = surv;
    uint32_t drs = 0;
    if (reuse) {
      dsize = surv_len;
    } else {
#pragma unroll
      for (int q = 0; q < K; ++q)
        if (q == drv) {
          dptr = nbr + S.pb[q] + rs[q];
          drs = rs[q];
        }
    }
    if (dsize == 0) {
      finish(A, i, S, j, false);
      return -1;
    }
    if (!A.step_multi[s]) {
      // single list: |S| = |range| - bound vertices inside it, pick by index
      uint32_t ex[K];
      uint32_t nex = 0;
#pragma unroll
      for (int q = 0; q < K; ++q) {
        ex[q] = INF;
        if (q < j && S.bnd[q] >= lo && S.bnd[q] < hi) {
          const uint32_t o = lb_thread(dptr, 0, dsize, S.bnd[q]);
          if (o < dsize && ldn(dptr, o) == S.bnd[q]) {
            ex[q] = o;
            ++nex;
          }
        }
      }
      const uint32_t cnt = dsize - nex;
      if (cnt == 0) {
        finish(A, i, S, j, false);
        return -1;
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
      S.alpha = __dmul_rn(S.alpha, (double)cnt);  // alpha *= |S_j| (ns_engine.cpp:39)
      const uint32_t pick = ldn(dptr, o);
#pragma unroll
      for (int q = 0; q < j; ++q)
        if (q == drv) {
          S.hbo[q] = drs + o + 1;
          S.hbl[q] = pick + 1;
        }
      bind(S, j, pick);
      continue;
    }
    // multi-list step: hand the intersection to the word-parallel phase
    IsectDesc<K> d;
    d.drv = dptr;
    d.dsize = dsize;
    d.lists = d.outs = d.core = 0;
    // a list whose owner is a core vertex is answered by one bit of the core
    // matrix for driver words inside the core; every driver element is >= lo,
    // so lo inside the core settles that for all words (bit 31), otherwise the
    // isect kernel checks each word's first element
    const bool use_core = A.g.core != nullptr;
#pragma unroll
    for (int q = 0; q < K - 1; ++q) {
      d.start[q] = 0;
      d.len[q] = 0;
      d.owner[q] = S.bnd[q];
      if (q < j && q != drv && (((in_m | out_m) >> q) & 1u)) {
        const bool is_out = (out_m >> q) & 1u;
        d.start[q] = is_out ? S.pb[q] : S.pb[q] + rs[q];
        d.len[q] = is_out ? S.pd[q] : re[q] - rs[q];
        d.lists |= 1u << q;
        if (is_out) d.outs |= 1u << q;
        if (use_core && S.bnd[q] >= A.g.core_base) d.core |= 1u << q;
      }
    }
    if (d.core && lo >= A.g.core_base) d.core |= 1u << 31;
    d.drv_pos = reuse ? NO_DRV : (uint32_t)drv;
    d.drv_rs = drs;
    if (local) {
      *local = d;
      return s;
    }
    reinterpret_cast<IsectDesc<K>*>(A.desc)[i] = d;
    A.work[i] = (dsize + 31) >> 5;
    store_state(A, i, S, j);
    return s;
  }
  finish(A, i, S, K, true);
  return -1;
}

template <int K>
__global__ void __launch_bounds__(256) fr_seed_kernel(const FrontierArgs A) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < A.count;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    Sample<K> S(A.seed, A.first_id + i);
    S.alpha = A.p.alpha0;
    const unsigned long long r0 = S.rng.next_below(A.g.arcs);  // ns_engine.cpp:29-33
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
    advance<K>(A, i, S, 0, nullptr, 0);
  }
}

// b ascending across lanes (INF padded); does any lane hold a?
__device__ __forceinline__ bool warp_contains(uint32_t b, uint32_t a) {
  int pos = 0;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const uint32_t t = __shfl_sync(FULL, b, pos + s - 1);
    if (t < a) pos += s;
  }
  return __shfl_sync(FULL, b, pos) == a;
}

// One warp per bitmap word; each warp walks a contiguous run of words. The run
// is consumed sample by sample: the owning sample is located once (k-ary over
// the word offsets, then 32 offsets per probe), its descriptor is read once
// into registers, and its words follow. Core lists cost one L2 word per lane;
// the rest load 32 splitters and finish with a short per-lane search.
template <int K>
__global__ void __launch_bounds__(256, 8) fr_isect_kernel(const FrontierArgs A, unsigned long long words) {
  const int lane = threadIdx.x & 31;
  const unsigned long long* __restrict__ off = A.offsets;
  const IsectDesc<K>* __restrict__ desc = reinterpret_cast<const IsectDesc<K>*>(A.desc);
  const uint32_t* __restrict__ nbr = A.g.nbr;
  const unsigned long long warp = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nwarps = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
  const unsigned long long per = (words + nwarps - 1) / nwarps;
  const unsigned long long w0 = warp * per, w1 = min(words, w0 + per);
  if (w0 >= w1) return;
  unsigned long long s;
  {  // last s with off[s] <= w0
    unsigned long long lo = 0, hi = A.count;
    while (hi - lo > 32) {
      const unsigned long long step = (hi - lo) / 33;
      const unsigned c = __popc(__ballot_sync(FULL, off[lo + (unsigned long long)(lane + 1) * step] <= w0));
      const unsigned long long nlo = c ? lo + c * step : lo;
      hi = c < 32 ? lo + (c + 1) * step : hi;
      lo = nlo;
    }
    const unsigned long long pos = lo + lane;
    s = lo + __popc(__ballot_sync(FULL, pos < hi && off[pos] <= w0)) - 1;
  }
  unsigned long long w = w0;
  while (w < w1) {
    // s = last sample with off[s] <= w (offsets are non-decreasing: a prefix test)
    for (;;) {
      const unsigned long long t = s + 1 + lane;
      const unsigned m = __ballot_sync(FULL, t <= A.count && off[t] <= w);
      s += __popc(m);
      if (m != FULL) break;
    }
    const unsigned long long we = min(w1, off[s + 1]);
    const IsectDesc<K>& d = desc[s];
    // loop-invariant scalars of the descriptor in registers; per-list fields stay in L1
    const uint32_t* __restrict__ drv = d.drv;
    const uint32_t dsize = d.dsize, lists = d.lists, outs = d.outs, core0 = d.core;
    const unsigned long long wbase = off[s];
    if (core0 == (lists | (1u << 31)) && outs == 0 && __popc(lists) <= 2) {
      // fast path (the common case on a relabelled graph): every other list is
      // a core row and the whole driver lies inside the core -> per word one
      // coalesced driver load and one bit probe per list
      const int q0 = __ffs(lists) - 1;
      const int q1 = __popc(lists) == 2 ? 31 - __clz(lists) : -1;
      const uint32_t cb = A.g.core_base;
      const uint32_t* r0 = A.g.core + (unsigned long long)(d.owner[q0] - cb) * A.g.core_wpr;
      const uint32_t* r1 = q1 >= 0 ? A.g.core + (unsigned long long)(d.owner[q1] - cb) * A.g.core_wpr : r0;
      for (; w < we; ++w) {
        const uint32_t o = (uint32_t)(w - wbase) * 32 + lane;
        bool fail = false;
        if (o < dsize) {
          const uint32_t c = ldo(drv, o) - cb;
          const uint32_t b0 = __ldg(r0 + (c >> 5));
          const uint32_t b1 = __ldg(r1 + (c >> 5));
          fail = !((b0 & b1) >> (c & 31) & 1u);
        }
        const unsigned bal = __ballot_sync(FULL, fail);
        if (lane == 0) A.bitmap[w] = bal;
      }
      continue;
    }
    for (; w < we; ++w) {
      const uint32_t o = (uint32_t)(w - wbase) * 32 + lane;
      const bool valid = o < dsize;
      const uint32_t a = valid ? ldo(drv, o) : INF;
      uint32_t core = core0;
      if (core && !(core >> 31) && __shfl_sync(FULL, a, 0) < A.g.core_base) core = 0;  // word leaves the core
      bool fail = false;
#pragma unroll
      for (int q = 0; q < K - 1; ++q) {
        if (!((lists >> q) & 1u)) continue;
        bool found;
        if ((core >> q) & 1u) {
          // a is inside the step's [lo, hi): membership in the restricted list is edge existence
          found = valid && core_has_edge(A.g, d.owner[q], a);
        } else {
          const uint32_t* B = nbr + d.start[q];
          const uint32_t nb = d.len[q];
          if (A.g.ehash) {
            found = valid && edge_lookup(A.g.ehash, A.g.ehash_mask, a, d.owner[q]);
          } else if (nb <= 32) {
            found = warp_contains((uint32_t)lane < nb ? ldo(B, (uint32_t)lane) : INF, a);
          } else {
            // 32 splitters at (i+1)*step; lane's bucket by shuffle search, then a short per-lane search
            const uint32_t step = nb / 33u;
            const uint32_t sp = ldo(B, (uint32_t)(lane + 1) * step);
            int c = 0;
#pragma unroll
            for (int sh = 16; sh >= 1; sh >>= 1) {
              const uint32_t t = __shfl_sync(FULL, sp, c + sh - 1);
              if (t < a) c += sh;
            }
            c += __shfl_sync(FULL, sp, c) < a ? 1 : 0;  // c = #splitters < a, in [0, 32]
            const uint32_t lo = c ? (uint32_t)c * step + 1 : 0;
            const uint32_t hi = c < 32 ? (uint32_t)(c + 1) * step : nb;
            const uint32_t at = lb_thread(B, lo, hi, a);
            found = at < nb && ldo(B, at) == a;
          }
        }
        fail = fail || (found == (bool)((outs >> q) & 1u));
      }
      const unsigned bal = __ballot_sync(FULL, valid && fail);
      if (lane == 0) A.bitmap[w] = bal;
    }
  }
}

// Thread per sample, warp-uniform loop structure so survivor compaction can use
// one atomic per warp.
template <int K>
__global__ void __launch_bounds__(256) fr_pick_kernel(const FrontierArgs A, int s_step) {
  const uint32_t* __restrict__ nbr = A.g.nbr;
  const int lane = threadIdx.x & 31;
  const int j = s_step + 2;
  const bool reuse_next = s_step + 1 < K - 2 && A.step_reuse[s_step + 1];
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long base = (blockIdx.x * (unsigned long long)blockDim.x) + (threadIdx.x & ~31u);
       base < A.count; base += stride) {
    const unsigned long long i = base + lane;
    const bool act = i < A.count && A.work[i] != 0;
    Sample<K> S(A.seed, A.first_id + (act ? i : 0));
    bool alive = false;
    uint32_t o_pick = 0, nsurv = 0, lo2 = 0, hi2 = INF, pick = 0;
    const IsectDesc<K>* dp = reinterpret_cast<const IsectDesc<K>*>(A.desc) + (act ? i : 0);
    const uint32_t* words = A.bitmap + (act ? A.offsets[i] : 0);
    uint32_t ex[K];
    uint32_t dsize = 0;
    if (act) {
      load_state(A, i, S, j);
      dsize = dp->dsize;
      const uint32_t* D = dp->drv;
      uint32_t lo, hi;
      step_bounds(A.p, s_step, S, lo, hi);
      // bound vertices that survived the intersection are not candidates (walker.hpp:70-82)
#pragma unroll
      for (int q = 0; q < K; ++q) {
        ex[q] = INF;
        if (q < j && S.bnd[q] >= lo && S.bnd[q] < hi) {
          const uint32_t o = lb_thread(D, 0, dsize, S.bnd[q]);
          if (o < dsize && ldn(D, o) == S.bnd[q] && !((words[o >> 5] >> (o & 31)) & 1u)) ex[q] = o;
        }
      }
      const uint32_t nw = (dsize + 31) >> 5;
      auto live = [&](uint32_t w) -> unsigned {
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
      } else {
        unsigned long long r = S.rng.next_below(cnt);
        for (uint32_t w = 0; w < nw; ++w) {
          const unsigned m = live(w);
          const unsigned pc = __popc(m);
          if (r < pc) {
            o_pick = w * 32 + __fns(m, 0, (int)r + 1);
            break;
          }
          r -= pc;
        }
        S.alpha = __dmul_rn(S.alpha, (double)cnt);  // alpha *= |S_j| (ns_engine.cpp:39)
        pick = ldn(D, o_pick);
        if (dp->drv_pos != NO_DRV) {
#pragma unroll
          for (int q = 0; q < K; ++q)
            if ((uint32_t)q == dp->drv_pos) {  // lower_bound(pick + 1) = drv_rs + o + 1
              S.hbo[q] = dp->drv_rs + o_pick + 1;
              S.hbl[q] = pick + 1;
            }
        }
        bind(S, j, pick);
        alive = true;
        if (reuse_next) {
          step_bounds(A.p, s_step + 1, S, lo2, hi2);
          for (uint32_t w = 0; w < nw; ++w) {
            unsigned m = live(w);
            while (m) {
              const uint32_t o = w * 32 + __ffs(m) - 1;
              m &= m - 1;
              const uint32_t x = ldn(D, o);
              nsurv += (o != o_pick && x >= lo2 && x < hi2) ? 1u : 0u;
            }
          }
        }
      }
    }
    // warp-aggregated allocation of the survivor lists
    uint32_t* surv = nullptr;
    if (reuse_next) {
      unsigned incl = nsurv;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned t = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += t;
      }
      unsigned long long wbase = 0;
      if (lane == 31 && incl) wbase = atomicAdd(A.surv_cursor + ((s_step + 1) & 1), (unsigned long long)incl);
      wbase = __shfl_sync(FULL, wbase, 31);
      const unsigned long long at = wbase + incl - nsurv;
      surv = A.survivors[(s_step + 1) & 1] + (at < A.surv_cap ? at : 0);
      if (alive && nsurv && at + nsurv <= A.surv_cap) {
        const uint32_t nw = (dsize + 31) >> 5;
        uint32_t k = 0;
        for (uint32_t w = 0; w < nw; ++w) {
          unsigned m = ~words[w];
          if (w == nw - 1 && (dsize & 31)) m &= (1u << (dsize & 31)) - 1u;
#pragma unroll
          for (int q = 0; q < K; ++q)
            if (ex[q] != INF && (ex[q] >> 5) == w) m &= ~(1u << (ex[q] & 31));
          while (m) {
            const uint32_t o = w * 32 + __ffs(m) - 1;
            m &= m - 1;
            const uint32_t x = ldn(dp->drv, o);
            if (o != o_pick && x >= lo2 && x < hi2) surv[k++] = x;
          }
        }
      }
    }
    if (alive) {
      if (reuse_next)
        advance<K>(A, i, S, s_step + 1, surv, nsurv);
      else
        advance<K>(A, i, S, s_step + 1, nullptr, 0);
    }
  }
}

// Fused sampler: one warp owns 32 samples (lane l <-> sample base + l).
// Scalar work (seed, bounds, ranges, driver choice, single-list steps) runs
// lane-parallel exactly as in fr_seed/fr_pick; each lane leaves its step
// descriptor in shared memory, and the warp then intersects the pending
// samples one after another, all 32 lanes on one sample's driver words (core
// bit tests or splitter searches, as in fr_isect), counts |S_j| from the live
// ballots, draws r with that sample's own CounterRng (broadcast, evaluated
// uniformly) and selects the r-th live element from the per-lane ballot words.
// No per-sample state leaves the SM between steps: no SoA state, scans,
// bitmaps or host round trips.
template <int K>
__device__ __forceinline__ unsigned live_word(const FrontierArgs& A, const IsectDesc<K>& d, uint32_t core, uint32_t w,
                                              int lane, int j) {
  const uint32_t* __restrict__ nbr = A.g.nbr;
  const uint32_t o = w * 32 + lane;
  const bool valid = o < d.dsize;
  const uint32_t a = valid ? ldo(d.drv, o) : INF;
  if (core && !(core >> 31) && __shfl_sync(FULL, a, 0) < A.g.core_base) core = 0;
  bool fail = !valid;
#pragma unroll
  for (int q = 0; q < K - 1; ++q) {
    if (q < j && a == d.owner[q]) fail = true;  // bound vertices are not candidates (walker.hpp:70-82)
    if (!((d.lists >> q) & 1u)) continue;
    bool found;
    if ((core >> q) & 1u) {
      found = valid && core_has_edge(A.g, d.owner[q], a);
    } else {
      const uint32_t* B = nbr + d.start[q];
      const uint32_t nb = d.len[q];
      if (nb <= 32) {
        found = warp_contains((uint32_t)lane < nb ? ldo(B, (uint32_t)lane) : INF, a);
      } else {
        const uint32_t step = nb / 33u;
        const uint32_t sp = ldo(B, (uint32_t)(lane + 1) * step);
        int c = 0;
#pragma unroll
        for (int sh = 16; sh >= 1; sh >>= 1) {
          const uint32_t t = __shfl_sync(FULL, sp, c + sh - 1);
          if (t < a) c += sh;
        }
        c += __shfl_sync(FULL, sp, c) < a ? 1 : 0;
        const uint32_t lo = c ? (uint32_t)c * step + 1 : 0;
        const uint32_t hi = c < 32 ? (uint32_t)(c + 1) * step : nb;
        const uint32_t at = lb_thread(B, lo, hi, a);
        found = at < nb && ldo(B, at) == a;
      }
    }
    fail = fail || (found == (bool)((d.outs >> q) & 1u));
  }
  return __ballot_sync(FULL, !fail);
}

template <int K>
__global__ void __launch_bounds__(256) fr_fused_kernel(const FrontierArgs A) {
  __shared__ IsectDesc<K> sdesc[256];
  const int lane = threadIdx.x & 31;
  IsectDesc<K>* wdesc = sdesc + (threadIdx.x & ~31u);
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long base = (blockIdx.x * (unsigned long long)blockDim.x) + (threadIdx.x & ~31u);
       base < A.count; base += stride) {
    const unsigned long long i = base + lane;
    const bool act = i < A.count;
    Sample<K> S(A.seed, A.first_id + (act ? i : 0));
    int pend = -1;
    if (act) {
      S.alpha = A.p.alpha0;
      const unsigned long long r0 = S.rng.next_below(A.g.arcs);  // ns_engine.cpp:29-33
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
      if (A.g.plain) {
        if (!swapped) {
          S.hbo[0] = (uint32_t)(r0 - S.pb[0]) + 1;
          S.hbl[0] = v + 1;
        } else {
          S.hbo[1] = (uint32_t)(r0 - S.pb[1]) + 1;
          S.hbl[1] = u + 1;
        }
      }
      pend = advance<K>(A, i, S, 0, nullptr, 0, wdesc + lane);
    }
    for (;;) {
      unsigned pending = __ballot_sync(FULL, pend >= 0);
      if (!pending) break;
      __syncwarp();
      bool picked = false;
      while (pending) {
        const int src = __ffs(pending) - 1;
        pending &= pending - 1;
        const int step = __shfl_sync(FULL, pend, src);
        const int j = step + 2;
        const IsectDesc<K>& d = wdesc[src];
        const uint32_t core = d.core;
        const uint32_t nw = (d.dsize + 31) >> 5;
        unsigned myword = 0;
        unsigned long long cnt = 0;
        for (uint32_t w = 0; w < nw; ++w) {
          const unsigned live = live_word<K>(A, d, core, w, lane, j);
          if ((uint32_t)lane == w) myword = live;
          cnt += __popc(live);
        }
        if (cnt == 0) {
          if (lane == src) {
            finish(A, i, S, j, false);
            pend = -1;
          }
          continue;
        }
        CounterRng rr(0);
        rr.key = __shfl_sync(FULL, S.rng.key, src);
        rr.ctr = __shfl_sync(FULL, S.rng.ctr, src);
        unsigned long long r = rr.next_below(cnt);  // uniform: every lane runs src's stream
        uint32_t o_pick = 0;
        if (nw <= 32) {
          const unsigned pc = __popc(myword);
          unsigned incl = pc;
#pragma unroll
          for (int dd = 1; dd < 32; dd <<= 1) {
            const unsigned t = __shfl_up_sync(FULL, incl, dd);
            if (lane >= dd) incl += t;
          }
          const unsigned excl = incl - pc;
          const unsigned who = __ballot_sync(FULL, excl <= r && r < incl);
          const int wl = __ffs(who) - 1;
          uint32_t ob = 0;
          if (lane == wl) ob = (uint32_t)wl * 32 + __fns(myword, 0, (int)(r - excl) + 1);
          o_pick = __shfl_sync(FULL, ob, wl);
        } else {  // long driver: replay the words up to the r-th live element
          for (uint32_t w = 0; w < nw; ++w) {
            const unsigned live = live_word<K>(A, d, core, w, lane, j);
            const unsigned pc = __popc(live);
            if (r < pc) {
              o_pick = w * 32 + __fns(live, 0, (int)r + 1);
              break;
            }
            r -= pc;
          }
        }
        const uint32_t pick = ldo(d.drv, o_pick);
        if (lane == src) {
          S.rng.ctr = rr.ctr;
          S.alpha = __dmul_rn(S.alpha, (double)cnt);  // alpha *= |S_j| (ns_engine.cpp:39)
          if (d.drv_pos != NO_DRV) {
#pragma unroll
            for (int q = 0; q < K; ++q)
              if ((uint32_t)q == d.drv_pos) {  // lower_bound(pick + 1) = drv_rs + o + 1
                S.hbo[q] = d.drv_rs + o_pick + 1;
                S.hbl[q] = pick + 1;
              }
          }
          bind(S, j, pick);
          picked = true;
        }
      }
      __syncwarp();
      if (picked) pend = advance<K>(A, i, S, pend + 1, nullptr, 0, wdesc + lane);
    }
  }
}

// Nested survivor reuse is exact but, at word granularity, rarely cheaper than
// re-intersecting (a sample's step-j driver is ~1 bitmap word either way) while
// compaction makes the pick phase divergent; off unless enabled.
bool g_frontier_reuse = false;

// step s can reuse step s-1's survivors when its lists and bounds nest
bool nests(const DevPlan& p, int s) {
  if (s == 0) return false;
  const unsigned pin = p.in_mask[s - 1], pout = p.out_mask[s - 1], in = p.in_mask[s], out = p.out_mask[s];
  if ((pin & in) != pin || (pout & out) != pout) return false;
  if (__builtin_popcount(pin) == 1 && pout == 0) return false;  // previous step was single-list
  const unsigned prev_pos = 1u << (s + 1);                         // position bound by step s-1
  const bool lo_ok = p.gt_mask[s - 1] == 0 || (p.gt_mask[s] & prev_pos) ||
                     (p.gt_mask[s] & p.gt_mask[s - 1]) == p.gt_mask[s - 1];
  const bool hi_ok = p.lt_mask[s - 1] == 0 || (p.lt_mask[s] & prev_pos) ||
                     (p.lt_mask[s] & p.lt_mask[s - 1]) == p.lt_mask[s - 1];
  return lo_ok && hi_ok;
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
    A.step_reuse[st] = g_frontier_reuse && A.step_multi[st] && nests(L.p, st);
  }
  const unsigned long long cap = std::min<unsigned long long>(L.count, kFrontierCap);
  A.cap = cap;
  size_t bytes = 0;
  auto carve = [&](size_t n) {
    size_t at = (bytes + 255) & ~size_t(255);
    bytes = at + n;
    return at;
  };
  const size_t o_ctr = carve(8 * cap), o_alpha = carve(8 * cap), o_bnd = carve(4ull * K * cap),
               o_hbo = carve(4ull * K * cap), o_hbl = carve(4ull * K * cap), o_work = carve(8 * (cap + 1)),
               o_off = carve(8 * (cap + 1)), o_desc = carve(sizeof(IsectDesc<K>) * cap), o_cur = carve(64);
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
  A.surv_cursor = reinterpret_cast<unsigned long long*>(slab + o_cur);
  void* tmp = slab + o_tmp;
  auto* h_total = static_cast<unsigned long long*>(ctx.get_pinned(2, 64));
  bool any_reuse = false;
  for (int st = 0; st < K - 2; ++st) any_reuse = any_reuse || A.step_reuse[st];

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
      const unsigned long long words = *h_total;
      if (words) {
        A.bitmap = static_cast<uint32_t*>(ctx.get(8, 4 * words + 64));
        if (any_reuse) {  // survivors <= driver elements <= 32 * words
          A.surv_cap = 32 * words;
          const int slot = (st + 1) & 1;
          A.survivors[slot] = static_cast<uint32_t*>(ctx.get(10 + slot, 4 * A.surv_cap + 64));
          AGPM_CUDA(cudaMemsetAsync(A.surv_cursor + slot, 0, 8, s));
        }
        const unsigned long long warps = std::min<unsigned long long>(words, (unsigned long long)sms * 64);
        fr_isect_kernel<K><<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(A, words);
        count_launch();
        AGPM_CUDA(cudaGetLastError());
      }
      fr_pick_kernel<K><<<blocks, 256, 0, s>>>(A, st);
      count_launch();
      AGPM_CUDA(cudaGetLastError());
    }
  }
}

template <int K>
void run_fused_k(const SampleLaunch& L, cudaStream_t s) {
  DeviceCtx& ctx = ctx_for_current_device();
  FrontierArgs A{};
  A.g = L.g;
  A.p = L.p;
  A.seed = L.seed;
  A.first_id = L.first_id;
  A.count = L.count;
  A.values = L.values;
  A.bindings = L.bindings;
  for (int st = 0; st < K - 2; ++st) {
    const unsigned in_m = L.p.in_mask[st], out_m = L.p.out_mask[st];
    A.step_multi[st] = !(__builtin_popcount(in_m) == 1 && out_m == 0);
    A.step_reuse[st] = 0;
  }
  static int occ = -1;
  if (occ < 0) {
    int o = 0;
    AGPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fr_fused_kernel<K>, 256, 0));
    occ = o > 0 ? o : 1;
  }
  const unsigned blocks =
      (unsigned)std::max<unsigned long long>(1, std::min<unsigned long long>((L.count + 255) / 256,
                                                                             (unsigned long long)ctx.sm_count * occ));
  fr_fused_kernel<K><<<blocks, 256, 0, s>>>(A);
  count_launch();
  AGPM_CUDA(cudaGetLastError());
}

}  // namespace

void set_frontier_reuse(bool on) { g_frontier_reuse = on; }

void launch_ns_fused(const SampleLaunch& L, cudaStream_t s) {
  if (L.bytes_out) throw std::invalid_argument("B_min accounting runs on the warp sampler");
  switch (L.p.k) {
    case 3: run_fused_k<3>(L, s); break;
    case 4: run_fused_k<4>(L, s); break;
    case 5: run_fused_k<5>(L, s); break;
    case 6: run_fused_k<6>(L, s); break;
    case 7: run_fused_k<7>(L, s); break;
    case 8: run_fused_k<8>(L, s); break;
    case 9: run_fused_k<9>(L, s); break;
    default: throw std::invalid_argument("device sampler needs 3 <= k <= 9");
  }
}

void launch_ns_frontier(const SampleLaunch& L, cudaStream_t s) {
  if (L.bytes_out) throw std::invalid_argument("B_min accounting runs on the warp sampler");
#define AGPM_K(KK)            \
  case KK:                    \
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
