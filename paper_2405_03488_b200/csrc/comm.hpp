// Rank communicators for the multi-GPU drivers.
//
// Two transports behind one handle:
//  * NCCL — one process per GPU (torchrun / MPI style). libnccl is opened with
//    dlopen on first use, so a process that already loaded NCCL (e.g. torch's
//    bundled copy) shares it, and single-GPU users never need it.
//  * local group — `world` ranks driven by host threads of ONE process (the
//    C++ drop-in's `workers` -> one host thread per GPU). Exchanges are
//    stream-synchronised peer copies between the ranks' device buffers behind a
//    host barrier; no kernel ever waits on another rank.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "agpm_b200.h"

namespace agpm_b200 {

int comm_rank(const agpm_comm* c);
int comm_world(const agpm_comm* c);
// recv[r * bytes .. (r+1) * bytes) = rank r's send buffer, for every rank (device buffers)
void comm_all_gather(agpm_comm* c, const void* d_send, void* d_recv, size_t bytes, cudaStream_t s);
// host-side barrier across the ranks (stream of the caller already synchronised)
void comm_barrier(agpm_comm* c, cudaStream_t s);

}  // namespace agpm_b200
