"""One-process-per-GPU plumbing for the sharded kernels.

The paper kernels shard along their natural independent dimension (rows of
softmax / rms_norm, the batch of bmm / conv2d / sdpa): every rank runs the
single-GPU kernel on its own shard, there is no collective on the data path,
timing is the max over ranks, and verification uses ONE gather of per-rank
error scalars after timing.  Works with NCCL (GPU) and gloo (CPU tests).
"""

from __future__ import annotations

import os


def world():
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(total: int, rank: int, world_size: int) -> tuple:
    """Contiguous, balanced [start, stop) of `total` units for `rank`."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad rank / world size")
    base, extra = divmod(total, world_size)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def _device_for(dist):
    import torch

    return torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend() == "nccl" else torch.device("cpu")


def max_over_ranks(x: float) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device_for(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_scalars(x: float) -> list:
    """The single verification collective: every rank's scalar, in rank order."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(x)]
    dev = _device_for(dist)
    bufs = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(dist.get_world_size())]
    dist.all_gather(bufs, torch.tensor([float(x)], dtype=torch.float64, device=dev))
    return [float(b.item()) for b in bufs]
