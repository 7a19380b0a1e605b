// Shared pieces of the sampling kernels (ns_lane.cu, ns_warp.cu, ns_frontier.cu, ns_lazy.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "device.cuh"
#include "rng.cuh"

namespace agpm_b200 {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kBallotWords = 64;  // shared ballots cover drivers up to 2048 elements

// Plan image on the device: per step, bitmasks over bound positions
// (in-lists, out-lists, greater_than and less_than of plan.hpp:21-29).
struct DevPlan {
  int k;
  int n_steps;
  int seed_ordered;
  int pad;
  double alpha0;  // seed_scale (plan.hpp:50-53): m or 2m
  unsigned short in_mask[AGPM_MAX_K - 2];
  unsigned short out_mask[AGPM_MAX_K - 2];
  unsigned short gt_mask[AGPM_MAX_K - 2];
  unsigned short lt_mask[AGPM_MAX_K - 2];
  // step s: after picking v_j (j = s + 2) from the list of bound position q, a
  // later step bounds N(v_j) by bnd[q] (e.g. the 4-cycle's S_3 = N(v0) ∩ N(v2)
  // > v1, with v2 picked from N(v1)): the twin arc of the pick then gives
  // lower_bound(bnd[q] + 1) in N(v_j) for free (core_bits.cu twin index)
  unsigned char twin_hint[AGPM_MAX_K - 2];
  // lazy verification (VerifyMode::Lazy, walker.hpp:56-62 / 88-107), positions
  int lazy;
  unsigned char tree_parent[AGPM_MAX_K - 2];
  unsigned char n_closure, n_terminal, n_nonadj;
  unsigned char closure[AGPM_MAX_PAIRS][2];   // edges not checked by a tree parent
  unsigned char terminal[AGPM_MAX_PAIRS][2];  // binding[a] < binding[b]
  unsigned char nonadj[AGPM_MAX_PAIRS][2];    // induced: must NOT be adjacent
};

struct GraphArgs {
  const VtxInfo* __restrict__ vtx;
  const uint32_t* __restrict__ nbr;
  const unsigned long long* __restrict__ seed_arcs;
  unsigned long long arcs;
  int plain;
  int loop_free;  // no vertex is in its own list (a single-list step's owner never needs a search)
  // dense-core adjacency bit matrix (core_bits.cu): bit (u - core_base, v - core_base)
  // of row-major rows of core_wpr words, for u, v >= core_base; null = off
  const uint32_t* __restrict__ core;
  uint32_t core_base;
  uint32_t core_wpr;
  // twin arcs (core_bits.cu): position of u in N(v) for arc (u -> v); null = off
  const uint32_t* __restrict__ twin;
  uint32_t n;  // vertices
};

// u, v >= core_base required
__device__ __forceinline__ bool core_has_edge(const GraphArgs& g, uint32_t u, uint32_t v) {
  const uint32_t c = v - g.core_base;
  return (__ldg(g.core + (unsigned long long)(u - g.core_base) * g.core_wpr + (c >> 5)) >> (c & 31)) & 1u;
}

struct SampleLaunch {
  GraphArgs g;
  DevPlan p;
  unsigned long long seed, first_id, count;
  double* values;
  uint32_t* bindings;             // nullable: count*k matching-order bindings
  unsigned long long* cursor;     // zeroed work counter
  unsigned long long* bytes_out;  // nullable: B_min accounting mode
};

__device__ __forceinline__ uint32_t ldn(const uint32_t* p, unsigned long long i) { return __ldg(p + i); }
// 32-bit element offset from a list base: one IMAD.WIDE.U32 per address
__device__ __forceinline__ uint32_t ldo(const uint32_t* p, uint32_t i) { return __ldg(p + i); }

__device__ __forceinline__ VtxInfo load_vtx(const VtxInfo* vtx, uint32_t v) {
  const int4 raw = __ldg(reinterpret_cast<const int4*>(vtx + v));
  VtxInfo vi;
  vi.begin = ((unsigned long long)(unsigned)raw.y << 32) | (unsigned)raw.x;
  vi.deg = (unsigned)raw.z;
  vi.up = (unsigned)raw.w;
  return vi;
}

// first index in [lo, hi) with nbr[i] >= x (hi if none)
__device__ __forceinline__ unsigned long long lower_bound_dev(const uint32_t* nbr, unsigned long long lo,
                                                              unsigned long long hi, uint32_t x) {
  while (lo < hi) {
    unsigned long long mid = (lo + hi) >> 1;
    if (ldn(nbr, mid) < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

constexpr uint32_t kNoVertex = 0xffffffffu;

// lower_bound of x within base[lo, hi] (answer in [lo, hi]); warp-uniform
// arguments, result uniform. `found` = (answer < hi && base[answer] == x).
__device__ __forceinline__ uint32_t kary_lb(const uint32_t* base, uint32_t lo, uint32_t hi, uint32_t x,
                                            int lane, bool* found) {
  const uint32_t end = hi;
  while (hi - lo > 32) {
    // 32 probes at lo + (i+1)*step, step = floor(span/33) >= 1, all < hi
    const uint32_t step = (hi - lo) / 33u;
    const unsigned bal = __ballot_sync(FULL, ldn(base, lo + (uint32_t)(lane + 1) * step) < x);
    const uint32_t c = __popc(bal);
    const uint32_t nlo = c ? lo + c * step + 1 : lo;
    hi = c < 32 ? lo + (c + 1) * step : hi;
    lo = nlo;
  }
  const uint32_t n = hi - lo;
  const uint32_t v = (uint32_t)lane < n ? ldn(base, lo + lane) : kNoVertex;
  const uint32_t r = lo + __popc(__ballot_sync(FULL, v < x));
  if (found) *found = r < end && ldn(base, r) == x;  // the answer may sit just past the last window
  return r;
}

// per-lane branchless lower_bound of a in base[0, n): the trip count depends
// only on n (warp-uniform), so lanes never diverge
__device__ __forceinline__ uint32_t lane_lb(const uint32_t* base, uint32_t n, uint32_t a) {
  if (n == 0) return 0;
  uint32_t b = 0;
  while (n > 1) {
    const uint32_t half = n >> 1;
    b = ldn(base, b + half - 1) < a ? b + half : b;
    n -= half;
  }
  return b + (ldn(base, b) < a ? 1u : 0u);
}

// b ascending across lanes (kNoVertex padded); does any lane hold a?
__device__ __forceinline__ bool chunk_contains(uint32_t b, uint32_t a) {
  int pos = 0;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const uint32_t t = __shfl_sync(FULL, b, pos + s - 1);
    if (t < a) pos += s;
  }
  return __shfl_sync(FULL, b, pos) == a;
}

// number of lanes whose b (ascending across lanes, kNoVertex padded) is < a
__device__ __forceinline__ uint32_t chunk_rank(uint32_t b, uint32_t a) {
  int pos = 0;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const uint32_t t = __shfl_sync(FULL, b, pos + s - 1);
    if (t < a) pos += s;
  }
  return (uint32_t)pos + (__shfl_sync(FULL, b, pos) < a ? 1u : 0u);
}

// 32-B sector span of u32 elements [a, b) (B_min model)
__device__ __forceinline__ unsigned long long sectors(unsigned long long a, unsigned long long b) {
  return b > a ? ((b * 4 - 1) >> 5) - ((a * 4) >> 5) + 1 : 0;
}

void launch_ns_lane(const SampleLaunch& L, cudaStream_t s);
void launch_ns_warp(const SampleLaunch& L, cudaStream_t s);
void launch_ns_frontier(const SampleLaunch& L, cudaStream_t s);
void launch_ns_lazy(const SampleLaunch& L, cudaStream_t s);
void launch_ns_flat(const SampleLaunch& L, cudaStream_t s, bool philox = false);
void set_frontier_reuse(bool on);

}  // namespace agpm_b200
