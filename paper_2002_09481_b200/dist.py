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
    """All-gather logits, all-reduce counts (SUM) and times (MAX).

    ``logits`` is (units, ...) per rank; ranks may hold different numbers of
    units (a 32-table sweep over 3 ranks: 11/11/10), so the unit counts are
    gathered first and every rank's block is padded to the largest for the
    one NCCL all-gather.  Returns (list of per-rank logits, counts, times); a
    no-op when torch.distributed is not initialised.
    """
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return [logits], counts, times
    world = dist.get_world_size(group)
    n = torch.tensor([logits.shape[0]], dtype=torch.int64, device=logits.device)
    sizes = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(v.item()) for v in sizes]
    top = max(sizes)
    pad = logits.new_zeros((top,) + tuple(logits.shape[1:]))
    pad[:logits.shape[0]] = logits
    gathered = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(gathered, pad.contiguous(), group=group)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(times, op=dist.ReduceOp.MAX, group=group)
    return [g[:k] for g, k in zip(gathered, sizes)], counts, times
