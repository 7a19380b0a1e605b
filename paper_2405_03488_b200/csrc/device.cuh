// Device-resident graph mirror and per-device runtime context.
//
// HBM layout of one view:
//   vtx[u]      16 B  {u64 begin, u32 degree, u32 up}: one 16-B load gives the
//                     list bounds and `up` = #neighbours <= u, so the upper
//                     suffix N+(u) = nbr[begin+up, begin+degree) is free.
//   nbr[]        4 B  per arc, lists ascending (reference layout).
//   seed_arcs[]  8 B  per view arc, (u << 32 | v) in arc-index order, so the
//                     uniform seed arc of ns_engine.cpp:12-23 is ONE gather
//                     instead of a log2(n) upper_bound over the prefix array.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <string>

#include "agpm_b200.h"
#include "common.hpp"

namespace agpm_b200 {

struct __align__(16) VtxInfo {
  unsigned long long begin;
  unsigned int deg;
  unsigned int up;
};

void cuda_check(cudaError_t e, const char* what);

// Every device neighbour array is followed by kNbrPad zeroed u32 so vector
// loads of a 16-B-aligned window around any list position stay in bounds.
constexpr uint64_t kNbrPad = 16;
uint32_t* alloc_nbr(uint64_t len, cudaStream_t s);
#define AGPM_CUDA(x) ::agpm_b200::cuda_check((x), #x)

struct DeviceCtx {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  // grow-only scratch
  void* scratch[16] = {nullptr};
  size_t scratch_bytes[16] = {0};
  void* pinned[4] = {nullptr};
  size_t pinned_bytes[4] = {0};
  void* get(int slot, size_t bytes);
  void* get_pinned(int slot, size_t bytes);
};

DeviceCtx& ctx_for_current_device();

// Device memory comes from the device's stream-ordered pool (release threshold
// unbounded): creating and dropping graph views, sparsified copies and
// scratch reuses cached memory instead of paying cudaMalloc/cudaFree each time.
// dev_malloc returns memory usable on any stream; dev_free keeps cudaFree's
// device-wide synchronisation.
cudaError_t dev_malloc_bytes(void** p, size_t bytes);
cudaError_t dev_free(void* p);
// stream-ordered free of a block only `s` has touched (no device-wide sync)
cudaError_t dev_free_stream(void* p, cudaStream_t s);
template <class T>
cudaError_t dev_malloc(T** p, size_t bytes) {
  return dev_malloc_bytes(reinterpret_cast<void**>(p), bytes);
}
cudaStream_t pick_stream(void* stream);
void count_launch(uint64_t n = 1);

// Makes `device` current for a scope (every call on a graph runs on the GPU
// that holds it, whatever device the calling thread had selected).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int device) {
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != device) {
      cuda_check(cudaSetDevice(device), "cudaSetDevice");
      prev = cur;
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// the plan is the edge-induced eager 4-cycle (k = 4, 4 edges, every vertex of degree 2)
bool plan_is_plain_4cycle(const agpm_plan* p);
// 4-cycles whose minimum vertex is < tau_id on a plain, symmetric, degree-relabelled
// view (cycle4_sparse.cu): the region split's C_sparse for the 4-cycle plan
unsigned long long cycle4_sparse_count(agpm_graph* g, uint32_t tau_id, cudaStream_t s);
}  // namespace agpm_b200

// C-ABI opaque handle
struct agpm_graph {
  int device = 0;
  uint32_t n = 0;
  uint64_t edge_count = 0;
  uint64_t arcs = 0;       // view arc total (seed space)
  uint64_t nbr_len = 0;
  uint64_t max_degree = 0;
  bool oriented = false;
  bool plain = true;       // end[u] == begin[u+1] and begin[0] == 0
  bool loop_free = false;  // no self-loops (checked when the view is built; ingest graphs by construction)
  agpm_b200::VtxInfo* vtx = nullptr;
  uint32_t* nbr = nullptr;
  unsigned long long* seed_arcs = nullptr;
  uint32_t* core = nullptr;  // dense-core bit matrix (core_bits.cu), built on demand
  uint32_t core_base = 0, core_wpr = 0, core_dim = 0;
  bool core_auto = false;  // core_dim was the auto choice (kept: the choice depends on free memory at build time)
  uint32_t* twin = nullptr;  // twin[i] = position of u in N(v) for arc i = (u -> v); plain views, on demand
  std::atomic<uint64_t> samples_drawn{0};  // ids sampled on this view by the flat / frontier samplers (twin index trigger)
  std::mutex index_mu;  // serialises the lazy index builds (core bits, twin arcs) of this view
  uint64_t bytes = 0;
};

namespace agpm_b200 {
// Build vtx / seed_arcs / arcs / max_degree for a view whose begin/end arrays
// already sit on the device (d_end may be null for plain views). Takes
// ownership of nothing; g->nbr must be set.
void finalize_view(agpm_graph* g, const unsigned long long* d_begin, const unsigned long long* d_end,
                   cudaStream_t s);
// build (or drop, when the configured dimension is 0) g->core for the current core dimension
void ensure_core_bits(agpm_graph* g, cudaStream_t s);
uint32_t core_dim_setting();
// build g->twin if absent (plain symmetric views): the seed arc then hints
// both seed lists
void ensure_twin_arcs(agpm_graph* g, cudaStream_t s);
// exact_count (exact_engine.cpp:66-91) on the device; root_limit keeps seeds whose
// first vertex is below it, shard/nshards keep every nshards-th 32-arc chunk
unsigned long long exact_count_device(const agpm_graph* g, const agpm_plan* plan, cudaStream_t s,
                                      uint32_t root_limit = 0xffffffffu, uint32_t shard = 0, uint32_t nshards = 1);
// the plan is the edge-induced eager 4-cycle (k = 4, 4 edges, every vertex of degree 2)
bool plan_is_plain_4cycle(const agpm_plan* p);
// 4-cycles whose minimum vertex is < tau_id on a plain, symmetric, degree-relabelled
// view (cycle4_sparse.cu): the region split's C_sparse for the 4-cycle plan
unsigned long long cycle4_sparse_count(agpm_graph* g, uint32_t tau_id, cudaStream_t s);
}  // namespace agpm_b200
