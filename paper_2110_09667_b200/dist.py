"""Host-side multi-process plumbing for libaa (one process per GPU).

Row partition (§4: "n/p contiguous rows", remainder to the leading
ranks, SPEC.md ShardLayout), rank discovery from the torchrun environment, the
max-over-ranks reduction used for timings, and the NCCL communicator handed to libaa.
No AA arithmetic here."""
from __future__ import annotations

import os


def rank_info():
    """(rank, world, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(n_global: int, rank: int, world: int) -> tuple[int, int]:
    """(offset, n_local) of this rank's contiguous row block."""
    if world < 1 or not (0 <= rank < world) or n_global < world:
        raise ValueError("need 0 <= rank < world <= n_global")
    base, rem = divmod(n_global, world)
    n_local = base + (1 if rank < rem else 0)
    offset = rank * base + min(rank, rem)
    return offset, n_local


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks of the default process group (identity if none)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def nccl_comm(group=None) -> int:
    """ncclComm_t of an (eagerly initialised) NCCL process group on the current device."""
    from . import aa
    return aa.torch_nccl_comm(group)
