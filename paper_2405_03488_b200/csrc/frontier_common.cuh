// Per-sample state, step descriptors and the lane-level step logic shared by
// the frontier (phase) sampler (ns_frontier.cu) and the on-chip samplers
// (flat: ns_flat.cu).
#pragma once

#include "ns_common.cuh"

namespace agpm_b200 {

namespace {

constexpr uint32_t INF = 0xffffffffu;
constexpr unsigned long long kFrontierCap = 1ull << 24;  // samples per pass
constexpr uint32_t NO_DRV = 0xffffffffu;

// Per-sample intersection job; other-list slots are indexed by matching position.
// Alignment: 16 B (vector loads in the frontier's global descriptor array) unless
// the including sampler asks otherwise (the flat sampler keeps them in shared memory).
// Twin hints for picked vertices (DevPlan::twin_hint) in the frontier phases: off.
// Measured per 2^24 4-cycle samples (the plan they target): RMAT-20 8.74 -> 8.95 ms,
// RMAT-22 13.39 -> 13.62 ms with them — N(v2)'s superset range already keeps it
// off the driver, so the exact range only costs the twin gather.
#ifndef AGPM_TWIN_HINT_SINGLE
#define AGPM_TWIN_HINT_SINGLE 0
#endif
#ifndef AGPM_DESC_ALIGN
#define AGPM_DESC_ALIGN 16
#endif
template <int K>
struct __align__(AGPM_DESC_ALIGN) IsectDesc {
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
  uint32_t exb;                       // bit q: bound vertex q lies inside the step's [lo, hi)
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
  // flat sampler: processing order of the launch's ids (nullptr = id order), see ns_flat.cu
  const uint32_t* order;
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

template <int K, class R = CounterRng>
struct Sample {
  uint32_t bnd[K], hbo[K], hbl[K];
  unsigned long long pb[K];
  uint32_t pd[K], up[K];
  bool loaded[K];
  R rng;
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

template <int K, class R>
__device__ __forceinline__ void ensure_vtx(const GraphArgs& g, Sample<K, R>& S, int q) {
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

template <int K, class R>
__device__ __forceinline__ uint32_t lbq(const uint32_t* nbr, Sample<K, R>& S, int q, uint32_t x, bool update) {
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

template <int K, class R>
__device__ __forceinline__ void bind(Sample<K, R>& S, int q, uint32_t v) {
#pragma unroll
  for (int t = 0; t < K; ++t)
    if (t == q) {
      S.bnd[t] = v;
      S.loaded[t] = false;
      S.hbl[t] = 0;  // "no dynamic hint": lower_bound(0) = 0 always holds
      S.hbo[t] = 0;
    }
}

template <int K, class R>
__device__ void store_state(const FrontierArgs& A, unsigned long long i, const Sample<K, R>& S, int nb) {
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

template <int K, class R>
__device__ void load_state(const FrontierArgs& A, unsigned long long i, Sample<K, R>& S, int nb) {
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

template <int K, class R>
__device__ void finish(const FrontierArgs& A, unsigned long long i, const Sample<K, R>& S, int nb, bool hit) {
  A.values[i] = hit ? S.alpha : 0.0;
  if (A.work) A.work[i] = 0;
  if (A.bindings) {
#pragma unroll
    for (int q = 0; q < K; ++q) A.bindings[i * K + q] = q < nb ? S.bnd[q] : INF;
  }
}

// order bounds of step s from the current bindings (walker.hpp:64-69)
template <int K, class R>
__device__ __forceinline__ void step_bounds(const DevPlan& p, int s, const Sample<K, R>& S, uint32_t& lo, uint32_t& hi) {
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
// once the sample is finished. With `local` set (flat kernel) the descriptor
// goes there and nothing is written to the SoA state.
template <int K, class R>
__device__ int advance(const FrontierArgs& A, unsigned long long i, Sample<K, R>& S, int s0, const uint32_t* surv,
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
        // the list's own owner is never in it on a loop-free graph: no search
        if (q < j && S.bnd[q] >= lo && S.bnd[q] < hi && !(A.g.loop_free && q == drv)) {
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
      uint32_t from = 0;
#pragma unroll
      for (int q = 0; q < j; ++q)
        if (q == drv) {
          S.hbo[q] = drs + o + 1;
          S.hbl[q] = pick + 1;
          from = S.bnd[q];
        }
      bind(S, j, pick);
      if (AGPM_TWIN_HINT_SINGLE && p.twin_hint[s] && A.g.twin && drv >= 0) {  // position of v_drv in N(pick)
        S.hbo[j] = __ldg(A.g.twin + (unsigned long long)(dptr - nbr) + o) + 1;
        S.hbl[j] = from + 1;
      }
      continue;
    }
    // multi-list step: hand the intersection to the word-parallel phase
    IsectDesc<K> d;
    d.drv = dptr;
    d.dsize = dsize;
    d.lists = d.outs = d.core = d.exb = 0;
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
      if (q < j && S.bnd[q] >= lo && S.bnd[q] < hi) d.exb |= 1u << q;
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
      // on-chip samplers keep the sample in registers across the intersection:
      // drop the cached vertex records (reloaded from vtx on the next step) so
      // they are not live there
#pragma unroll
      for (int q = 0; q < K; ++q) S.loaded[q] = false;
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

template <int K>
__device__ __forceinline__ unsigned live_word_g(const GraphArgs& g, const IsectDesc<K>& d, uint32_t core, uint32_t w,
                                                int lane, int j) {
  const uint32_t* __restrict__ nbr = g.nbr;
  const uint32_t o = w * 32 + lane;
  const bool valid = o < d.dsize;
  const uint32_t a = valid ? ldo(d.drv, o) : INF;
  if (core && !(core >> 31) && __shfl_sync(FULL, a, 0) < g.core_base) core = 0;
  bool fail = !valid;
#pragma unroll
  for (int q = 0; q < K - 1; ++q) {
    if (q < j && a == d.owner[q]) fail = true;  // bound vertices are not candidates (walker.hpp:70-82)
    if (!((d.lists >> q) & 1u)) continue;
    bool found;
    if ((core >> q) & 1u) {
      found = valid && core_has_edge(g, d.owner[q], a);
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
__device__ __forceinline__ unsigned live_word(const FrontierArgs& A, const IsectDesc<K>& d, uint32_t core, uint32_t w,
                                              int lane, int j) {
  return live_word_g<K>(A.g, d, core, w, lane, j);
}

}  // namespace

}  // namespace agpm_b200
