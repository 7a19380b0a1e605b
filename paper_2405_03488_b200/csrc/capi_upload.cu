// agpm_graph_upload_host: host CsrGraph -> device view (needs both handle types).
#include "device.cuh"
#include "host_graph.hpp"

extern "C" int agpm_graph_upload_host(const agpm_host_graph* g, void* stream, agpm_graph** out) {
  if (!g) {
    agpm_b200::set_last_error("null argument");
    return AGPM_E_INVALID;
  }
  return agpm_graph_upload(g->g.n, g->g.edge_count, g->g.offsets.data(), nullptr, g->g.neighbors.data(),
                           g->g.neighbors.size(), g->g.oriented, stream, out);
}

extern "C" int agpm_host_graph_pin(agpm_host_graph* g) {
  return agpm_b200::guarded([&] {
    if (!g) throw std::invalid_argument("null argument");
    if (g->pinned) return;
    agpm_b200::ctx_for_current_device();
    if (!g->g.offsets.empty())
      AGPM_CUDA(cudaHostRegister(g->g.offsets.data(), 8 * g->g.offsets.size(), cudaHostRegisterDefault));
    if (!g->g.neighbors.empty())
      AGPM_CUDA(cudaHostRegister(g->g.neighbors.data(), 4 * g->g.neighbors.size(), cudaHostRegisterDefault));
    g->pinned = true;
  });
}

void agpm_b200_unpin_host_graph(agpm_host_graph* g) {
  if (g && g->pinned) {
    if (!g->g.offsets.empty()) cudaHostUnregister(g->g.offsets.data());
    if (!g->g.neighbors.empty()) cudaHostUnregister(g->g.neighbors.data());
    g->pinned = false;
  }
}
