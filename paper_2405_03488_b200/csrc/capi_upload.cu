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
