"""Host-side logic of the one-process-per-GPU runs (bench.py --gpus N).

HyRes of one cube is a global computation (the Gram and the periodised DWT
couple all pixels), so the multi-GPU path shards INDEPENDENT cubes across ranks
(BASELINE.json configs[4]: "a batch of 64 independent 256x256x191 cubes
distributed data-parallel over 8 GPUs") with no data-path
collective.  This module holds only that plumbing -- which cubes a rank owns and
how rank timings combine -- so the gloo tests exercise exactly what the bench
runs.  It contains none of the method's arithmetic.
"""
from __future__ import annotations

import os
from typing import List, Tuple


def env_rank() -> Tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(n_units: int, rank: int, world: int) -> List[int]:
    """Units (cube indices / seeds) owned by `rank`: round-robin, so every unit is
    owned by exactly one rank and the per-rank counts differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return list(range(rank, n_units, world))


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar (a timing) over the process group; identity when
    torch.distributed is not initialised.  The bench reports the MAX over ranks."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def whole_job_rate(units_total: float, seconds_max: float) -> float:
    """Whole-job throughput: units processed by ALL ranks / the slowest rank's time."""
    if seconds_max <= 0:
        raise ValueError("non-positive time")
    return units_total / seconds_max
