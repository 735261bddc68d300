"""Multi-GPU plumbing for the GNS step (one process per GPU).

The job's d*t*p ranks are block-mapped onto the N physical GPUs (SURVEY §8e:
"fewer physical GPUs than d*t*p: virtual ranks are block-mapped").  Every
physical rank reduces its virtual ranks' buckets into its own N+1 fp64 slots
(device), then ONE collective — an NCCL all-reduce of those N+1 scalars over
NVLink (Alg. 1 AllReduce) — gives every rank the whole-job
s_n and gbar^2, and the finalize kernel runs redundantly on each rank.
torch.distributed is used only to broadcast the NCCL unique id and for
barriers; the data-path collective is the library's own NCCL communicator.
"""
from __future__ import annotations

from typing import Sequence


def block_map(job_ranks: int, world: int, rank: int) -> list[int]:
    """Virtual (job) ranks hosted by physical `rank` of `world`: a contiguous
    block, so model-parallel neighbours stay on one GPU."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if job_ranks % world:
        raise ValueError(f"{job_ranks} job ranks do not block-map onto {world} GPUs")
    per = job_ranks // world
    return list(range(rank * per, (rank + 1) * per))


def share_unique_id(dist, make_id, rank: int) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank receives it."""
    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def slot_of(coords: Sequence[int], micro: int, M: int) -> int:
    """Accumulator slot of (i_d, m): s_{i_d, m} lives at i_d * M + m."""
    return coords[0] * M + micro


def attach(gns_device, dist, world: int, rank: int) -> None:
    """Give a GnsDevice its NCCL communicator (no-op on one GPU)."""
    if world <= 1:
        return
    from .device import nccl_unique_id
    uid = share_unique_id(dist, nccl_unique_id, rank)
    gns_device.attach_nccl(world, rank, uid)


def attach_p2p(gns_device, dist, world: int, rank: int) -> list:
    """Give a GnsDevice NVLink mailboxes for allreduce_finalize_p2p: each
    rank allocates its mailbox, the CUDA IPC handles are all-gathered over
    torch.distributed, the peers' mailboxes are mapped.  Returns the base
    pointers to pass to device.ipc_close when done."""
    from .device import ipc_handle_ptr, ipc_open
    mine = gns_device.mailbox(world)
    handles = [None] * world
    dist.all_gather_object(handles, ipc_handle_ptr(mine))
    peers, bases = [], []
    for q in range(world):
        if q == rank:
            peers.append(mine)
        else:
            p, b = ipc_open(handles[q], gns_device.device)
            peers.append(p)
            bases.append(b)
    gns_device.attach_mailboxes(world, rank, peers)
    dist.barrier()
    return bases
