"""Multi-GPU plumbing: one process per GPU, torch.distributed for the
handshake only.

The data path never goes through torch.distributed or NCCL: every GPU's
worker rows are exported as CUDA IPC handles, exchanged once here, and the
library's kernels then load/store peer rows directly over NVLink/NVSwitch
(two-shot ordered fold) with flag barriers in peer memory.
"""
from __future__ import annotations

import os
from typing import List, Optional


def pin_host_cores(local_rank: int, local_world: int) -> list:
    """Give each GPU's process its own host cores (an equal, disjoint share
    of this process's CPU set; no-op with fewer than two cores per rank).
    The small-row step is host-launch-latency sensitive: two ranks' launch
    loops time-sharing one core make it up to 2x slower in an unlucky run.
    Returns the cores now in use."""
    cpus = sorted(os.sched_getaffinity(0))
    k = len(cpus) // max(1, local_world)
    if local_world > 1 and k >= 2:
        mine = cpus[local_rank * k:(local_rank + 1) * k]
        os.sched_setaffinity(0, mine)
        return mine
    return cpus


def exchange_handles(engine, group=None) -> List[bytes]:
    """all_gather every rank's IPC handle blob (rank order)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    blobs: List[Optional[bytes]] = [None] * world
    dist.all_gather_object(blobs, engine.ipc_export(), group=group)
    for i, b in enumerate(blobs):
        if not isinstance(b, (bytes, bytearray)):
            raise RuntimeError(f"rank {i} sent no IPC handle")
    return [bytes(b) for b in blobs]


def attach(engine, group=None) -> None:
    """Map every peer's rows into this context (collective: call on all ranks)."""
    import torch.distributed as dist
    if dist.get_world_size(group) != engine.n_gpus:
        raise ValueError("process group size must equal the engine's n_gpus")
    if dist.get_rank(group) != engine.rank:
        raise ValueError("engine rank must equal the process rank")
    engine.ipc_attach(exchange_handles(engine, group))


def local_slice(world_size: int, n_gpus: int, rank: int) -> range:
    """Global worker ranks hosted by GPU `rank` (contiguous packing, gpu(k) = k / P)."""
    if world_size % n_gpus:
        raise ValueError("world_size must be a multiple of n_gpus")
    per = world_size // n_gpus
    return range(rank * per, (rank + 1) * per)
