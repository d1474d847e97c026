"""torch.distributed plumbing for multi-process (one GPU per rank) runs.

torch.distributed is only the bootstrap/control channel: the step's data
path uses the library's own NCCL communicator, created from a ncclUniqueId
that rank 0 generates and these helpers broadcast.
"""
from __future__ import annotations

import os

from .api import ClusterConfig, Transport, nccl_unique_id


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


def share_nccl_id(dist) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank returns the same 128 bytes."""
    obj = [nccl_unique_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def nccl_config(base: ClusterConfig, dist, device: int) -> ClusterConfig:
    """ClusterConfig for this rank: worker id = rank, K = world size, NCCL transport."""
    base.workers = dist.get_world_size()
    base.transport = Transport.NCCL
    base.rank = dist.get_rank()
    base.device = device
    base.nccl_id = share_nccl_id(dist)
    return base


def max_over_ranks(dist, value: float, device="cpu") -> float:
    """Max of a scalar over ranks (step times are reported as the slowest rank)."""
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
