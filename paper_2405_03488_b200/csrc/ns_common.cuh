// Shared pieces of the two sampling kernels (ns_lane.cu, ns_warp.cu).
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
};

struct GraphArgs {
  const VtxInfo* __restrict__ vtx;
  const uint32_t* __restrict__ nbr;
  const unsigned long long* __restrict__ seed_arcs;
  unsigned long long arcs;
  int plain;
  const unsigned long long* __restrict__ ehash;  // edge table (frontier sampler)
  uint32_t ehash_mask;
};

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

// 32-B sector span of u32 elements [a, b) (B_min model)
__device__ __forceinline__ unsigned long long sectors(unsigned long long a, unsigned long long b) {
  return b > a ? ((b * 4 - 1) >> 5) - ((a * 4) >> 5) + 1 : 0;
}

void launch_ns_lane(const SampleLaunch& L, cudaStream_t s);
void launch_ns_warp(const SampleLaunch& L, cudaStream_t s);
void launch_ns_frontier(const SampleLaunch& L, cudaStream_t s);
void set_frontier_reuse(bool on);

}  // namespace agpm_b200
