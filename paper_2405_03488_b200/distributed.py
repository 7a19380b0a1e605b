"""Process setup for the multi-GPU drivers.

The sharded drivers are native (csrc/ns_device.cu online_loop, csrc/comm.cu):
the CSR is replicated on every GPU, global sample id i always uses
CounterRng(seed, 0, i), and per round rank r draws the r-th block of ids
(agpm_ns_shard_round), folds it into 1000-sample window records, the records
are all-gathered over NCCL (rank order = id order) and every rank runs the
single-GPU stop test on them — so an N-rank run stops at the 1-rank (=
reference workers = 1) n with the same hits and sums. This module only turns a
torchrun process into a rank: device selection from LOCAL_RANK and the NCCL
unique-id handshake (rank 0 creates it, torch.distributed broadcasts the 128
bytes). Only moments cross ranks; nothing here is on the sampling path.
"""
import os

__all__ = ["env_rank", "nccl_comm"]


def env_rank():
    """(rank, world, local_rank) from the torchrun environment (1-rank defaults)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def nccl_comm(dist, rank, world):
    """The product's NCCL communicator for this rank (agpm_comm_init_nccl); `dist`
    is an initialised torch.distributed (any backend) used for the id handshake.
    Call with this rank's GPU current."""
    from . import Comm, nccl_unique_id

    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return Comm.nccl(rank, world, obj[0])
