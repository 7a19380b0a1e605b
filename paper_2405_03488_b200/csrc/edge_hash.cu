// Build of the device edge-membership table (edge_hash.cuh).
#include <algorithm>

#include "device.cuh"
#include "edge_hash.cuh"

namespace agpm_b200 {
namespace {

__device__ bool try_bucket(unsigned long long* table, unsigned long long b, unsigned long long key) {
  for (int s = 0; s < 4; ++s) {
    const unsigned long long prev = atomicCAS(table + 4 * b + s, kEmptyKey, key);
    if (prev == kEmptyKey || prev == key) return true;
  }
  return false;
}

// one thread per arc; each undirected edge is inserted from its u < v arc
__global__ void edge_hash_build_kernel(const unsigned long long* __restrict__ arcs, unsigned long long n_arcs,
                                       unsigned long long* table, uint32_t mask, unsigned int* overflow) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n_arcs;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long arc = arcs[i];
    const uint32_t u = (uint32_t)(arc >> 32), v = (uint32_t)arc;
    if (u >= v) continue;
    const unsigned long long key = arc;  // u << 32 | v with u < v
    if (try_bucket(table, mix64(key) & mask, key)) continue;
    if (try_bucket(table, mix64(key ^ kHash2Salt) & mask, key)) continue;
    atomicAdd(overflow, 1u);
  }
}

}  // namespace

void ensure_edge_hash(agpm_graph* g, cudaStream_t s) {
  if (g->ehash) return;
  DeviceCtx& ctx = ctx_for_current_device();
  const unsigned long long edges = std::max<unsigned long long>(g->arcs / 2, 1);
  unsigned long long buckets = 1;
  while (buckets * 2 < edges) buckets <<= 1;  // load factor <= 1/2 over 4-slot buckets
  buckets <<= 1;
  auto* overflow = static_cast<unsigned int*>(ctx.get(3, 64));
  for (int attempt = 0; attempt < 4; ++attempt, buckets <<= 1) {
    if (buckets > (1ull << 32)) throw std::invalid_argument("edge hash: too many edges");
    unsigned long long* table = nullptr;
    AGPM_CUDA(dev_malloc(&table, 32ull * buckets));
    AGPM_CUDA(cudaMemsetAsync(table, 0xff, 32ull * buckets, s));
    AGPM_CUDA(cudaMemsetAsync(overflow, 0, 4, s));
    const unsigned blocks = (unsigned)std::min<unsigned long long>((g->arcs + 255) / 256, (unsigned long long)ctx.sm_count * 16);
    if (g->arcs) {
      edge_hash_build_kernel<<<blocks ? blocks : 1, 256, 0, s>>>(g->seed_arcs, g->arcs, table,
                                                                  (uint32_t)(buckets - 1), overflow);
      count_launch();
      AGPM_CUDA(cudaGetLastError());
    }
    unsigned int h_over = 0;
    AGPM_CUDA(cudaMemcpyAsync(&h_over, overflow, 4, cudaMemcpyDeviceToHost, s));
    AGPM_CUDA(cudaStreamSynchronize(s));
    if (h_over == 0) {
      g->ehash = table;
      g->ehash_mask = (uint32_t)(buckets - 1);
      g->bytes += 32ull * buckets;
      return;
    }
    AGPM_CUDA(dev_free(table));
  }
  throw cuda_error("edge hash build kept overflowing");
}

}  // namespace agpm_b200
