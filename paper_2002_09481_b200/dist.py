"""Multi-GPU plumbing: shard independent units, exchange results once.

The path shards with no data-path collective:

* range-batches -- quantization ranges are per batch (graph.py:270-275), so
  each batch is a self-contained unit; rank g takes batches g, g+G, ...
* candidate truth tables (the multiplier sweep, config 4) -- each table is an
  independent network; rank g takes tables g, g+G, ...

The only collective is after the timed work: ``exchange_results`` all-gathers
the logits (NCCL over NVLink on the GPU box; gloo in the CPU tests) and
all-reduces the agreement counts and the per-rank device times (MAX).
"""

from __future__ import annotations

import torch


def shard(n_units: int, world: int, rank: int) -> list[int]:
    """Round-robin units for this rank (batches or candidate tables)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    return list(range(rank, n_units, world))


def exchange_results(logits: torch.Tensor, counts: torch.Tensor, times: torch.Tensor, group=None):
    """All-gather logits (equal shapes per rank), all-reduce counts (SUM) and times (MAX).

    Returns (gathered_logits [world x ...], counts, times); a no-op when
    torch.distributed is not initialised.
    """
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return logits.unsqueeze(0), counts, times
    world = dist.get_world_size(group)
    gathered = [torch.empty_like(logits) for _ in range(world)]
    dist.all_gather(gathered, logits.contiguous(), group=group)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(times, op=dist.ReduceOp.MAX, group=group)
    return torch.stack(gathered), counts, times
