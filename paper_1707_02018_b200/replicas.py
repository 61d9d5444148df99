"""Host-side rank logic for running the hot path on N GPUs as independent replicas.

DESIGN.md §8: the images of a batch are independent for W, W*, W-dagger, R, R* and grad f
(SURVEY.md §8(e)), so N GPUs run N replicas with no data-path collective.  The process
group is used only for the barrier that brackets the timed region and for the
max-over-ranks of the device time.  Everything here is backend-agnostic (nccl on the GPU
box, gloo in the CPU tests) and holds none of the method's arithmetic.
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass(frozen=True)
class RankInfo:
    world: int
    rank: int
    local: int


def rank_info() -> RankInfo:
    """WORLD_SIZE / RANK / LOCAL_RANK from the torchrun environment (1 / 0 / 0 without it)."""
    return RankInfo(int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
                    int(os.environ.get("LOCAL_RANK", "0")))


def shard(n_units: int, world: int, rank: int) -> range:
    """Contiguous share of n_units independent units (images) owned by `rank`.

    The first n_units % world ranks get one extra unit; shares are disjoint and cover
    [0, n_units) exactly (an empty range is a valid share)."""
    if world < 1 or not 0 <= rank < world or n_units < 0:
        raise ValueError(f"bad shard request n={n_units} world={world} rank={rank}")
    base, extra = divmod(n_units, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def _device_for(backend: str):
    import torch
    return torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")


def barrier(world: int) -> None:
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(value: float, world: int) -> float:
    """Max of a per-rank scalar (the device time of the timed region) over all ranks."""
    if world == 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device_for(dist.get_backend()))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, world: int) -> float:
    """Sum of a per-rank count (units processed) over all ranks."""
    if world == 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device_for(dist.get_backend()))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def whole_job_rate(units_per_rank: float, seconds_per_rank: float, world: int) -> float:
    """value = units all ranks processed / max-over-ranks time (the bench contract)."""
    total = sum_over_ranks(units_per_rank, world)
    t = max_over_ranks(seconds_per_rank, world)
    return total / t
