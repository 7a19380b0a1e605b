// Device graph mirror (CsrView on HBM), per-device context, misc C-ABI.
#include <cub/cub.cuh>

#include <atomic>
#include <unordered_map>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <sys/syscall.h>
#include <unistd.h>
#include <vector>

#include "device.cuh"

namespace agpm_b200 {

namespace {
thread_local std::string t_err;
std::atomic<uint64_t> g_launches{0};
std::mutex g_ctx_mu;
bool g_pool_ready[64] = {false};
}  // namespace

void set_last_error(const std::string& msg) { t_err = msg; }

// Large blocks (32 MB .. 1 GB) freed by dev_free are parked here, up to 4 GB per
// process, and handed back to the next dev_malloc of the same size: recreating a
// graph view (the e2e loop) then reuses its buffers outright. The stream-ordered
// pool alone periodically took 20-55 ms to hand back the 512 MB core matrix.
namespace {
struct Parked {
  void* p;
  size_t bytes;
  int device;
};
std::mutex g_park_mu;
std::vector<Parked> g_parked;
std::unordered_map<void*, std::pair<size_t, int>> g_big;  // live large blocks -> (size, owning device)
size_t g_parked_bytes = 0;
constexpr size_t kParkMin = 32ull << 20, kParkMax = 1ull << 30, kParkCap = 4ull << 30;
}  // namespace

cudaError_t dev_malloc_bytes(void** p, size_t bytes) {
  DeviceCtx& ctx = ctx_for_current_device();
  if (bytes >= kParkMin && bytes <= kParkMax) {
    std::lock_guard<std::mutex> lk(g_park_mu);
    for (size_t i = 0; i < g_parked.size(); ++i)
      if (g_parked[i].bytes == bytes && g_parked[i].device == ctx.device) {
        *p = g_parked[i].p;
        g_parked_bytes -= bytes;
        g_parked.erase(g_parked.begin() + (long)i);
        g_big[*p] = {bytes, ctx.device};
        return cudaSuccess;
      }
  }
  cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 1, ctx.stream);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(ctx.stream);
  if (e == cudaSuccess && bytes >= kParkMin && bytes <= kParkMax) {
    std::lock_guard<std::mutex> lk(g_park_mu);
    g_big[*p] = {bytes, ctx.device};
  }
  return e;
}

cudaError_t dev_free(void* p) {
  if (!p) return cudaSuccess;
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return e;
  DeviceCtx& ctx = ctx_for_current_device();
  {
    std::lock_guard<std::mutex> lk(g_park_mu);
    auto it = g_big.find(p);
    if (it != g_big.end()) {
      const size_t bytes = it->second.first;
      const int owner = it->second.second;  // parked under the GPU that holds it
      g_big.erase(it);
      if (g_parked_bytes + bytes <= kParkCap) {  // idle (device synchronised above): reusable at once
        g_parked.push_back({p, bytes, owner});
        g_parked_bytes += bytes;
        return cudaSuccess;
      }
    }
  }
  return cudaFreeAsync(p, ctx.stream);
}
// Free a block only stream `s` has used (temporaries of a view build): stream-
// ordered, no device-wide synchronisation — a view upload on one host thread
// then never waits for sampling kernels another thread runs meanwhile.
cudaError_t dev_free_stream(void* p, cudaStream_t s) {
  if (!p) return cudaSuccess;
  size_t bytes = 0;
  int owner = 0;
  {
    std::lock_guard<std::mutex> lk(g_park_mu);
    auto it = g_big.find(p);
    if (it != g_big.end()) {
      bytes = it->second.first;
      owner = it->second.second;
      g_big.erase(it);
    }
  }
  if (bytes) {  // a parkable block: park once the stream is done with it
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_park_mu);
    if (g_parked_bytes + bytes <= kParkCap) {
      g_parked.push_back({p, bytes, owner});
      g_parked_bytes += bytes;
      return cudaSuccess;
    }
  }
  return cudaFreeAsync(p, s);
}

void count_launch(uint64_t n) { g_launches += n; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
      throw nodevice_error(std::string("no usable CUDA device (the B200 path has no CPU fallback): ") +
                           cudaGetErrorString(e));
    throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
  }
}

void* DeviceCtx::get(int slot, size_t bytes) {
  if (scratch_bytes[slot] < bytes) {
    if (scratch[slot]) AGPM_CUDA(dev_free(scratch[slot]));
    size_t grow = bytes + bytes / 4;
    AGPM_CUDA(dev_malloc(&scratch[slot], grow));
    scratch_bytes[slot] = grow;
  }
  return scratch[slot];
}

uint32_t* alloc_nbr(uint64_t len, cudaStream_t s) {
  uint32_t* p = nullptr;
  AGPM_CUDA(dev_malloc(&p, 4ull * (len + kNbrPad)));
  AGPM_CUDA(cudaMemsetAsync(p + len, 0, 4ull * kNbrPad, s));
  return p;
}

void* DeviceCtx::get_pinned(int slot, size_t bytes) {
  if (pinned_bytes[slot] < bytes) {
    if (pinned[slot]) AGPM_CUDA(cudaFreeHost(pinned[slot]));
    AGPM_CUDA(cudaMallocHost(&pinned[slot], bytes));
    pinned_bytes[slot] = bytes;
  }
  return pinned[slot];
}

// One context (stream + scratch) per host thread and device: host threads
// driving ranks of a local group — several may share a GPU — never share
// scratch buffers or the library stream. A worker thread's contexts are
// released when it exits; the main thread's live until process exit.
namespace {
struct ThreadCtxs {
  DeviceCtx* c[64] = {nullptr};
  ~ThreadCtxs() {
    if (static_cast<pid_t>(syscall(SYS_gettid)) == getpid()) return;  // main thread: process teardown
    for (int d = 0; d < 64; ++d) {
      DeviceCtx* x = c[d];
      if (!x) continue;
      if (cudaSetDevice(d) == cudaSuccess) {
        cudaStreamSynchronize(x->stream);
        for (void* p : x->scratch)
          if (p) dev_free(p);
        for (void* p : x->pinned)
          if (p) cudaFreeHost(p);
        cudaStreamDestroy(x->stream);
      }
      delete x;
    }
  }
};
thread_local ThreadCtxs t_ctx;
}  // namespace

DeviceCtx& ctx_for_current_device() {
  int dev = 0;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw nodevice_error("no CUDA device visible: the B200 sampling path has no CPU fallback");
  AGPM_CUDA(cudaGetDevice(&dev));
  if (!t_ctx.c[dev]) {
    auto* c = new DeviceCtx();
    c->device = dev;
    AGPM_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, dev));
    AGPM_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    {
      std::lock_guard<std::mutex> lk(g_ctx_mu);
      if (!g_pool_ready[dev]) {
        cudaMemPool_t pool;
        AGPM_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t keep = ~0ull;  // never trim: freed graph memory stays cached for the next view
        AGPM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        // never make an allocation on one stream wait for work pending on another
        // (a view uploaded on one host thread must not queue behind the sampling
        // kernels of another); reuse only what is already free
        int no = 0;
        AGPM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no));
        g_pool_ready[dev] = true;
      }
    }
    t_ctx.c[dev] = c;
  }
  return *t_ctx.c[dev];
}

cudaStream_t pick_stream(void* stream) {
  return stream ? static_cast<cudaStream_t>(stream) : ctx_for_current_device().stream;
}

namespace {

__global__ void vtx_kernel(const unsigned long long* __restrict__ begin,
                           const unsigned long long* __restrict__ end, const uint32_t* __restrict__ nbr,
                           uint32_t n, VtxInfo* __restrict__ vtx, unsigned long long* __restrict__ deg,
                           unsigned long long* __restrict__ loops) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long b = begin[u];
    unsigned long long e = end ? end[u] : begin[u + 1];
    // up = #neighbours <= u  (lower_bound of u+1)
    unsigned long long lo = b, hi = e;
    while (lo < hi) {
      unsigned long long mid = (lo + hi) >> 1;
      if (nbr[mid] <= (uint32_t)u)
        lo = mid + 1;
      else
        hi = mid;
    }
    if (lo > b && nbr[lo - 1] == (uint32_t)u) atomicOr(loops, 1ull);  // a self-loop u-u
    VtxInfo v;
    v.begin = b;
    v.deg = (unsigned int)(e - b);
    v.up = (unsigned int)(lo - b);
    vtx[u] = v;
    deg[u] = e - b;
  }
}

// one warp per vertex: seed_arcs[prefix[u] + j] = u<<32 | nbr[begin[u] + j]
__global__ void seed_arcs_kernel(const VtxInfo* __restrict__ vtx, const uint32_t* __restrict__ nbr,
                                 const unsigned long long* __restrict__ prefix, uint32_t n,
                                 unsigned long long* __restrict__ arcs) {
  const int lane = threadIdx.x & 31;
  uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t u = w; u < n; u += nw) {
    VtxInfo v = vtx[u];
    unsigned long long base = prefix[u];
    unsigned long long hi = (unsigned long long)u << 32;
    for (unsigned int j = lane; j < v.deg; j += 32) arcs[base + j] = hi | nbr[v.begin + j];
  }
}

}  // namespace

void finalize_view(agpm_graph* g, const unsigned long long* d_begin, const unsigned long long* d_end,
                   cudaStream_t s) {
  const uint32_t n = g->n;
  DeviceCtx& ctx = ctx_for_current_device();
  AGPM_CUDA(dev_malloc(&g->vtx, sizeof(VtxInfo) * (size_t)(n ? n : 1)));
  unsigned long long* deg = nullptr;
  unsigned long long* prefix = nullptr;
  AGPM_CUDA(dev_malloc(&deg, sizeof(unsigned long long) * ((size_t)n + 1)));
  AGPM_CUDA(dev_malloc(&prefix, sizeof(unsigned long long) * ((size_t)n + 1)));
  unsigned long long* red = nullptr;
  AGPM_CUDA(dev_malloc(&red, 2 * sizeof(unsigned long long)));  // [0] max degree, [1] self-loop flag
  AGPM_CUDA(cudaMemsetAsync(red + 1, 0, sizeof(unsigned long long), s));
  int blocks = ctx.sm_count * 8;
  if (n) {
    vtx_kernel<<<blocks, 256, 0, s>>>(d_begin, d_end, g->nbr, n, g->vtx, deg, red + 1);
    count_launch();
    AGPM_CUDA(cudaGetLastError());
  }
  AGPM_CUDA(cudaMemsetAsync(prefix, 0, sizeof(unsigned long long), s));
  AGPM_CUDA(cudaMemsetAsync(deg + n, 0, sizeof(unsigned long long), s));
  size_t tmp_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, deg, prefix + 1, (int64_t)n, s);
  size_t tmp_bytes2 = 0;
  cub::DeviceReduce::Max(nullptr, tmp_bytes2, deg, red, (int64_t)n + 1, s);
  void* tmp = ctx.get(7, std::max(tmp_bytes, tmp_bytes2) + 16);
  if (n) {
    AGPM_CUDA(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, deg, prefix + 1, (int64_t)n, s));
  }
  unsigned long long arcs = 0, maxd = 0;
  AGPM_CUDA(cudaMemcpyAsync(&arcs, prefix + n, sizeof(arcs), cudaMemcpyDeviceToHost, s));
  AGPM_CUDA(cub::DeviceReduce::Max(tmp, tmp_bytes2, deg, red, (int64_t)n + 1, s));
  AGPM_CUDA(cudaMemcpyAsync(&maxd, red, sizeof(maxd), cudaMemcpyDeviceToHost, s));
  unsigned long long loops = 0;
  AGPM_CUDA(cudaMemcpyAsync(&loops, red + 1, sizeof(loops), cudaMemcpyDeviceToHost, s));
  AGPM_CUDA(cudaStreamSynchronize(s));
  g->arcs = arcs;
  g->max_degree = maxd;
  g->loop_free = loops == 0;
  AGPM_CUDA(dev_malloc(&g->seed_arcs, sizeof(unsigned long long) * (size_t)(arcs ? arcs : 1)));
  if (n && arcs) {
    seed_arcs_kernel<<<blocks, 256, 0, s>>>(g->vtx, g->nbr, prefix, n, g->seed_arcs);
    count_launch();
    AGPM_CUDA(cudaGetLastError());
  }
  AGPM_CUDA(cudaStreamSynchronize(s));
  AGPM_CUDA(dev_free_stream(deg, s));
  AGPM_CUDA(dev_free_stream(prefix, s));
  AGPM_CUDA(dev_free_stream(red, s));
  g->bytes = sizeof(VtxInfo) * (uint64_t)n + 4ull * g->nbr_len + 8ull * arcs;
}

}  // namespace agpm_b200

using namespace agpm_b200;

extern "C" {

const char* agpm_last_error(void) { return t_err.c_str(); }
int agpm_version(void) { return AGPM_B200_ABI_VERSION; }
uint64_t agpm_kernel_launches(void) { return g_launches.load(); }

int agpm_device_count(int* n) {
  return guarded([&] {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    *n = e == cudaSuccess ? c : 0;
  });
}

int agpm_set_device(int device) {
  return guarded([&] { AGPM_CUDA(cudaSetDevice(device)); });
}

int agpm_current_device(void) {
  int d = -1;
  if (cudaGetDevice(&d) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return d;
}

int agpm_sync(void* stream) {
  return guarded([&] { AGPM_CUDA(cudaStreamSynchronize(pick_stream(stream))); });
}

int agpm_graph_upload(uint32_t n, uint64_t edge_count, const uint64_t* begin, const uint64_t* end,
                      const uint32_t* neighbors, uint64_t neighbor_len, int oriented, void* stream,
                      agpm_graph** out) {
  return guarded([&] {
    if (!begin || !out || (neighbor_len && !neighbors)) throw std::invalid_argument("null argument");
    DeviceCtx& ctx = ctx_for_current_device();
    cudaStream_t s = pick_stream(stream);
    auto* g = new agpm_graph();
    g->device = ctx.device;
    g->n = n;
    g->edge_count = edge_count;
    g->oriented = oriented != 0;
    g->nbr_len = neighbor_len;
    g->plain = end == nullptr && begin[0] == 0;
    unsigned long long *d_begin = nullptr, *d_end = nullptr;
    size_t nb = end ? n : (size_t)n + 1;
    AGPM_CUDA(dev_malloc(&d_begin, sizeof(uint64_t) * (nb ? nb : 1)));
    AGPM_CUDA(cudaMemcpyAsync(d_begin, begin, sizeof(uint64_t) * nb, cudaMemcpyHostToDevice, s));
    if (end) {
      AGPM_CUDA(dev_malloc(&d_end, sizeof(uint64_t) * (n ? n : 1)));
      AGPM_CUDA(cudaMemcpyAsync(d_end, end, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, s));
    }
    g->nbr = alloc_nbr(neighbor_len, s);
    if (neighbor_len)
      AGPM_CUDA(cudaMemcpyAsync(g->nbr, neighbors, sizeof(uint32_t) * neighbor_len,
                                cudaMemcpyHostToDevice, s));
    finalize_view(g, d_begin, d_end, s);
    if (!g->loop_free) {  // the device samplers assume simple graphs (as every builder here produces)
      AGPM_CUDA(dev_free_stream(d_begin, s));
      if (d_end) AGPM_CUDA(dev_free_stream(d_end, s));
      AGPM_CUDA(cudaStreamSynchronize(s));
      agpm_graph_free(g);
      throw std::invalid_argument("the graph has self-loops; build it with CsrGraph::from_edges (which drops them)");
    }
    AGPM_CUDA(dev_free_stream(d_begin, s));
    if (d_end) AGPM_CUDA(dev_free_stream(d_end, s));
    AGPM_CUDA(cudaStreamSynchronize(s));  // the view is complete when the call returns
    *out = g;
  });
}

int agpm_graph_free(agpm_graph* g) {
  return guarded([&] {
    if (!g) return;
    DeviceGuard guard(g->device);  // free (and park) on the GPU that holds the view
    dev_free(g->vtx);
    dev_free(g->nbr);
    dev_free(g->seed_arcs);
    if (g->core) dev_free(g->core);
    if (g->twin) dev_free(g->twin);
    delete g;
  });
}

int agpm_graph_info(const agpm_graph* g, uint32_t* n, uint64_t* edge_count, uint64_t* arcs,
                    int* oriented, uint64_t* device_bytes) {
  return guarded([&] {
    if (n) *n = g->n;
    if (edge_count) *edge_count = g->edge_count;
    if (arcs) *arcs = g->arcs;
    if (oriented) *oriented = g->oriented;
    if (device_bytes) *device_bytes = g->bytes;
  });
}

int agpm_graph_max_degree(const agpm_graph* g, uint64_t* out) {
  return guarded([&] {
    if (!g || !out) throw std::invalid_argument("null argument");
    *out = g->max_degree;
  });
}

int agpm_graph_neighbor_len(const agpm_graph* g, uint64_t* len) {
  return guarded([&] {
    if (!g || !len) throw std::invalid_argument("null argument");
    *len = g->nbr_len;
  });
}

int agpm_graph_download(const agpm_graph* g, uint64_t* begin, uint64_t* end, uint32_t* neighbors) {
  return guarded([&] {
    std::vector<VtxInfo> v(g->n);
    AGPM_CUDA(cudaMemcpy(v.data(), g->vtx, sizeof(VtxInfo) * g->n, cudaMemcpyDeviceToHost));
    for (uint32_t u = 0; u < g->n; ++u) {
      if (begin) begin[u] = v[u].begin;
      if (end) end[u] = v[u].begin + v[u].deg;
    }
    if (neighbors && g->nbr_len)
      AGPM_CUDA(cudaMemcpy(neighbors, g->nbr, 4 * g->nbr_len, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
