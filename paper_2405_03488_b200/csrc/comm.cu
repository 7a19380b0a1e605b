// Rank communicators (NCCL over NVLink/NVSwitch, or an in-process thread group)
// and the sharded exact count. See comm.hpp.
#include <dlfcn.h>
#include <nccl.h>  // types and enums only; the symbols come from dlopen

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "comm.hpp"
#include "device.cuh"

struct agpm_comm_group {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t phase = 0;
  std::vector<const void*> send;
  std::vector<int> device;
  int members = 0;  // live agpm_comm handles (the group is freed with the last one)
};

struct agpm_comm {
  int rank = 0, world = 1, device = 0;
  bool nccl = false;
  ncclComm_t nc = nullptr;
  agpm_comm_group* group = nullptr;
};

namespace agpm_b200 {
namespace {

// ------------------------------------------------------------ NCCL, resolved at run time
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static std::once_flag once;
  static NcclApi api;
  static std::string why;
  std::call_once(once, [] {
    // an already-loaded libnccl (same soname, e.g. torch's) is reused
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      why = dlerror();
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.init_rank = reinterpret_cast<decltype(api.init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!api.get_unique_id || !api.init_rank || !api.all_gather || !api.all_reduce || !api.destroy)
    throw cuda_error("NCCL is not available in this process: " + (why.empty() ? std::string("missing symbols") : why));
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const NcclApi& a = nccl();
    throw cuda_error(std::string(what) + ": " + (a.error_string ? a.error_string(r) : "NCCL error"));
  }
}

// host barrier of a local group; `publish` runs under the lock before arriving
template <class F>
void group_barrier(agpm_comm_group* g, F&& publish) {
  std::unique_lock<std::mutex> lk(g->mu);
  publish();
  const uint64_t my_phase = g->phase;
  if (++g->arrived == g->world) {
    g->arrived = 0;
    ++g->phase;
    g->cv.notify_all();
  } else {
    g->cv.wait(lk, [&] { return g->phase != my_phase; });
  }
}

}  // namespace

int comm_rank(const agpm_comm* c) { return c->rank; }
int comm_world(const agpm_comm* c) { return c->world; }

void comm_all_gather(agpm_comm* c, const void* d_send, void* d_recv, size_t bytes, cudaStream_t s) {
  if (c->world == 1) {
    if (d_send != d_recv) AGPM_CUDA(cudaMemcpyAsync(d_recv, d_send, bytes, cudaMemcpyDeviceToDevice, s));
    return;
  }
  if (c->nccl) {
    nccl_check(nccl().all_gather(d_send, d_recv, bytes, ncclUint8, c->nc, s), "ncclAllGather");
    return;
  }
  // local group: every rank's send buffer is complete before it is published
  AGPM_CUDA(cudaStreamSynchronize(s));
  agpm_comm_group* g = c->group;
  group_barrier(g, [&] {
    g->send[c->rank] = d_send;
    g->device[c->rank] = c->device;
  });
  for (int r = 0; r < c->world; ++r)
    AGPM_CUDA(cudaMemcpyPeerAsync(static_cast<char*>(d_recv) + (size_t)r * bytes, c->device, g->send[r],
                                  g->device[r], bytes, s));
  AGPM_CUDA(cudaStreamSynchronize(s));
  group_barrier(g, [] {});  // nobody reuses its send buffer while a peer still copies it
}

void comm_barrier(agpm_comm* c, cudaStream_t s) {
  if (c->world == 1) return;
  if (c->nccl) {  // a one-word all-reduce doubles as a barrier
    DeviceCtx& ctx = ctx_for_current_device();
    auto* w = static_cast<unsigned long long*>(ctx.get(11, 64));
    nccl_check(nccl().all_reduce(w, w, 1, ncclUint64, ncclSum, c->nc, s), "ncclAllReduce");
    AGPM_CUDA(cudaStreamSynchronize(s));
    return;
  }
  AGPM_CUDA(cudaStreamSynchronize(s));
  group_barrier(c->group, [] {});
}

}  // namespace agpm_b200

using namespace agpm_b200;

extern "C" {

int agpm_nccl_unique_id(unsigned char id[AGPM_NCCL_ID_BYTES]) {
  return guarded([&] {
    static_assert(sizeof(ncclUniqueId) == AGPM_NCCL_ID_BYTES, "ncclUniqueId size");
    if (!id) throw std::invalid_argument("null argument");
    ncclUniqueId u;
    nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

int agpm_comm_init_nccl(int rank, int world, const unsigned char id[AGPM_NCCL_ID_BYTES], agpm_comm** out) {
  return guarded([&] {
    if (!id || !out) throw std::invalid_argument("null argument");
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("rank must be in [0, world)");
    DeviceCtx& ctx = ctx_for_current_device();
    auto* c = new agpm_comm();
    c->rank = rank;
    c->world = world;
    c->device = ctx.device;
    c->nccl = true;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    try {
      nccl_check(nccl().init_rank(&c->nc, world, u, rank), "ncclCommInitRank");
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int agpm_comm_group_create(int world, agpm_comm_group** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null argument");
    if (world < 1) throw std::invalid_argument("world must be >= 1");
    auto* g = new agpm_comm_group();
    g->world = world;
    g->send.assign(world, nullptr);
    g->device.assign(world, 0);
    *out = g;
  });
}

int agpm_comm_init_local(agpm_comm_group* group, int rank, agpm_comm** out) {
  return guarded([&] {
    if (!group || !out) throw std::invalid_argument("null argument");
    if (rank < 0 || rank >= group->world) throw std::invalid_argument("rank must be in [0, world)");
    DeviceCtx& ctx = ctx_for_current_device();
    auto* c = new agpm_comm();
    c->rank = rank;
    c->world = group->world;
    c->device = ctx.device;
    c->group = group;
    {
      std::lock_guard<std::mutex> lk(group->mu);
      ++group->members;
    }
    *out = c;
  });
}

int agpm_comm_group_free(agpm_comm_group* group) {
  return guarded([&] {
    if (!group) return;
    {
      std::lock_guard<std::mutex> lk(group->mu);
      if (group->members != 0) throw std::invalid_argument("comm group still has live communicators");
    }
    delete group;
  });
}

int agpm_comm_free(agpm_comm* c) {
  return guarded([&] {
    if (!c) return;
    if (c->nccl && c->nc) nccl().destroy(c->nc);
    if (c->group) {
      std::lock_guard<std::mutex> lk(c->group->mu);
      --c->group->members;
    }
    delete c;
  });
}

int agpm_comm_info(const agpm_comm* c, int* rank, int* world, int* device, int* is_nccl) {
  return guarded([&] {
    if (!c) throw std::invalid_argument("null argument");
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
    if (device) *device = c->device;
    if (is_nccl) *is_nccl = c->nccl ? 1 : 0;
  });
}

int agpm_comm_all_gather_dev(agpm_comm* c, const void* d_send, void* d_recv, uint64_t bytes_per_rank,
                             void* stream) {
  return guarded([&] {
    if (!c || (bytes_per_rank && (!d_send || !d_recv))) throw std::invalid_argument("null argument");
    DeviceGuard dg(c->device);
    comm_all_gather(c, d_send, d_recv, bytes_per_rank, pick_stream(stream));
  });
}

int agpm_exact_count_sharded(agpm_comm* c, agpm_graph* g, const agpm_plan* plan, uint64_t* count, void* stream) {
  // exact_count (exact_engine.cpp:66-91) split over the ranks: rank r counts the
  // seeds of 32-arc chunks r, r + world, ... and the u64 partials are gathered
  // and summed (integer, so the order is immaterial)
  return guarded([&] {
    if (!c || !g || !plan || !count) throw std::invalid_argument("null argument");
    DeviceGuard dg(g->device);
    DeviceCtx& ctx = ctx_for_current_device();
    cudaStream_t s = pick_stream(stream);
    const unsigned long long mine = exact_count_device(g, plan, s, 0xffffffffu, (uint32_t)c->rank, (uint32_t)c->world);
    auto* d = static_cast<unsigned long long*>(ctx.get(11, 8ull * (c->world + 1)));
    AGPM_CUDA(cudaMemcpyAsync(d + c->world, &mine, 8, cudaMemcpyHostToDevice, s));
    comm_all_gather(c, d + c->world, d, 8, s);
    std::vector<unsigned long long> all(c->world);
    AGPM_CUDA(cudaMemcpyAsync(all.data(), d, 8ull * c->world, cudaMemcpyDeviceToHost, s));
    AGPM_CUDA(cudaStreamSynchronize(s));
    unsigned long long total = 0;
    for (unsigned long long x : all) total += x;
    *count = total;
  });
}

}  // extern "C"
