"""Stream sharding across the GPUs of one node.

Camera streams are independent reference ``Network`` instances
(/root/reference/proj/SPEC.md:370; per-stream state cbconv.hpp:65-79), so the
multi-GPU path partitions STREAMS over ranks and never exchanges data: global
stream g runs on rank g mod world. The only collectives are the timing
barrier and the max-over-ranks reduction of the timed region (bench.py);
both go through ``torch.distributed`` (nccl on the GPU box, gloo in the CPU
tests), so this module is backend-agnostic.
"""
from __future__ import annotations

from typing import List


def streams_for_rank(streams_per_rank: int, rank: int, world: int) -> List[int]:
    """Global stream ids owned by ``rank`` under weak scaling: every rank runs
    ``streams_per_rank`` streams, stream g lives on rank g % world."""
    if world < 1 or not (0 <= rank < world) or streams_per_rank < 0:
        raise ValueError(f"bad shard request: S={streams_per_rank} rank={rank} world={world}")
    return [rank + world * s for s in range(streams_per_rank)]


def stream_seed(global_stream: int) -> int:
    """Clip seed of a global stream (distinct per stream; stream 0 -> seed 1)."""
    return global_stream + 1


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the timed region's device milliseconds) over
    all ranks; identity when torch.distributed is not initialised."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier() -> None:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def aggregate_rate(world: int, units_per_rank: int, ms_max: float) -> float:
    """Whole-job throughput: the units all ranks processed / the slowest rank's time."""
    return world * units_per_rank / (ms_max / 1000.0)


def gather_objects(obj):
    """Per-rank values (e.g. each rank's sampled clocks) collected on every
    rank, rank order; [obj] when torch.distributed is not initialised."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out
