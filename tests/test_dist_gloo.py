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
    logits = torch.full((4, 3), float(rank)) + torch.arange(3.0)
    counts = torch.tensor([rank + 1, 4], dtype=torch.int64)
    times = torch.tensor([10.0 * (rank + 1), 1.0], dtype=torch.float64)
    g, c, t = exchange_results(logits, counts, times)
    q.put((rank, units, g.tolist(), c.tolist(), t.tolist()))
    dist.destroy_process_group()


def test_shard_round_robin_covers_all_units_once():
    for world in (1, 2, 3, 8):
        seen = sorted(u for r in range(world) for u in shard(32, world, r))
        assert seen == list(range(32))
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def test_exchange_results_two_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, units, g, c, t in res:
        assert units == list(range(rank, 10, 2))
        assert len(g) == 2 and g[0][0] == [0.0, 1.0, 2.0] and g[1][0] == [1.0, 2.0, 3.0]
        assert c == [3, 8]
        assert t == [20.0, 1.0]


def test_exchange_is_noop_single_process():
    lg = torch.zeros(2, 3)
    g, c, t = exchange_results(lg, torch.tensor([1]), torch.tensor([2.0]))
    assert g.shape == (1, 2, 3) and c.tolist() == [1] and t.tolist() == [2.0]
