"""Multi-GPU plumbing (one process per GPU; torch.distributed for rendezvous only).

The PQR data path never goes through torch.distributed: the library owns an NCCL
communicator created from a 128-byte ncclUniqueId (``pqr_nccl_unique_id`` on rank 0,
broadcast here as a Python object), and issues its own collectives (CholQR2: one
allgather of the (k+s) x s Gram per pass; TSQR: one allgather of the GPU roots'
(C+s) x s blocks per call).  Rows are sharded contiguously; the last
shard absorbs the remainder.
"""
from __future__ import annotations

import os


def row_shard(n_global: int, world: int, rank: int) -> tuple[int, int]:
    """(offset, n_local) of `rank`'s contiguous row shard of n_global rows."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base = n_global // world
    off = rank * base
    n_local = base + (n_global - base * world if rank == world - 1 else 0)
    return off, n_local


def env_rank_world():
    """(rank, world, local_rank) from the torchrun environment (defaults: single process)."""
    if "RANK" not in os.environ:
        return 0, 1, 0
    return int(os.environ["RANK"]), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def init(backend: str, device=None):
    """init_process_group from the environment (MASTER_ADDR defaults to 127.0.0.1)."""
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if dist.is_initialized():
        return
    kw = {}
    if device is not None and backend == "nccl":
        kw["device_id"] = device
    dist.init_process_group(backend, **kw)


def broadcast_bytes(payload: bytes | None, src: int = 0) -> bytes:
    """Broadcast a small byte string (e.g. the NCCL unique id) from `src` to every rank."""
    import torch.distributed as dist

    obj = [payload if dist.get_rank() == src else None]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def nccl_id_for_library(world: int) -> bytes | None:
    """Rank 0 creates the library's ncclUniqueId and every rank receives it (None if world == 1)."""
    if world == 1:
        return None
    import torch.distributed as dist

    from . import pqr

    mine = pqr.pqr_nccl_unique_id() if dist.get_rank() == 0 else None
    return broadcast_bytes(mine)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a host scalar over all ranks (timings: the job is as slow as its slowest rank)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allgather_fixed_order_sum(local, device=None):
    """Sum of every rank's array in rank order (the bitwise-reproducible reduction the library
    performs on its allgathered Gram blocks).  Used by tests and host-side checks."""
    import numpy as np
    import torch
    import torch.distributed as dist

    t = torch.as_tensor(np.ascontiguousarray(local), dtype=torch.float64, device=device)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    acc = parts[0].clone()
    for p in parts[1:]:
        acc += p
    return acc.cpu().numpy(), [p.cpu().numpy() for p in parts]
