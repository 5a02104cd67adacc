"""World-size-2 gloo test of the multi-GPU plumbing (sharding + the single result exchange)."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2002_09481_b200.dist import exchange_results, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    units = shard(10, world, rank)
    # one (units, 3) logits block per rank; shard(10, 3, r) is uneven: 4 / 3 / 3 units
    logits = torch.full((len(units), 3), float(rank)) + torch.arange(3.0)
    counts = torch.tensor([rank + 1, 4], dtype=torch.int64)
    times = torch.tensor([10.0 * (rank + 1), 1.0], dtype=torch.float64)
    g, c, t = exchange_results(logits, counts, times)
    q.put((rank, units, [x.tolist() for x in g], c.tolist(), t.tolist()))
    dist.destroy_process_group()


def test_shard_round_robin_covers_all_units_once():
    for world in (1, 2, 3, 8):
        seen = sorted(u for r in range(world) for u in shard(32, world, r))
        assert seen == list(range(32))
    with pytest.raises(ValueError):
        shard(4, 2, 2)


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_results_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, units, g, c, t in res:
        assert units == list(range(rank, 10, world))
        assert len(g) == world
        for r in range(world):  # every rank's block, trimmed to its own unit count
            assert len(g[r]) == len(range(r, 10, world))
            assert all(row == [float(r), r + 1.0, r + 2.0] for row in g[r])
        assert c == [sum(range(1, world + 1)), 4 * world]
        assert t == [10.0 * world, 1.0]


def test_exchange_is_noop_single_process():
    lg = torch.zeros(2, 3)
    g, c, t = exchange_results(lg, torch.tensor([1]), torch.tensor([2.0]))
    assert len(g) == 1 and g[0].shape == (2, 3) and c.tolist() == [1] and t.tolist() == [2.0]
