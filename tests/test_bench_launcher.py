"""bench.py's multi-rank launcher on CPU: --gpus N re-launches under torch.distributed.run (gloo, --stub)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _bench(*args, timeout=300):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                           "MASTER_PORT")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, env=env, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-3000:]
    lines = []
    for ln in out.stdout.splitlines():
        try:
            obj = json.loads(ln)
        except ValueError:
            continue
        if isinstance(obj, dict) and "metric" in obj:
            lines.append(obj)
    return lines


@pytest.mark.parametrize("world,per_rank", [(2, [16, 16]), (3, [11, 11, 10])])
def test_sweep_sharded_over_launched_ranks(world, per_rank):
    """All 32 candidate tables covered exactly once, uneven shards counted from the gathered lists."""
    lines = _bench("--gpus", str(world), "--stub", "--workload", "r62sweep", "--steps", "2", "--warmup", "3",
                   "--batch", "8")
    assert len(lines) == 1, lines  # rank 0 alone prints
    ln = lines[0]
    assert ln["n_gpus"] == world
    assert ln["units"]["per_rank"] == per_rank and ln["units"]["total"] == 32 and ln["units"]["covered_once"]
    assert ln["scaling"] == "strong" and ln["steps"] == 2 and ln["warmup"] == 3
    # images = batch x networks x steps over all ranks; value = GMAC/s over the max-over-ranks time
    macs = ln["config"]["macs_per_image"]
    t = ln["ms_per_step"] * ln["steps"] / 1e3
    assert abs(ln["value"] - 8 * 32 * 2 * macs / t / 1e9) / ln["value"] < 1e-3
    assert ln["logits_gathered"] == [world]


def test_range_batches_two_ranks():
    lines = _bench("--gpus", "2", "--stub", "--workload", "r8", "--steps", "2", "--batch", "16")
    assert len(lines) == 1
    ln = lines[0]
    assert ln["n_gpus"] == 2 and ln["scaling"] == "weak"
    assert ln["units"] == {"kind": "range-batches", "per_rank": [1, 1], "total": 2, "covered_once": True}
    assert "dp2" in ln["config"]["parallelism"]


def test_single_process_stub_unchanged():
    lines = _bench("--stub", "--workload", "r8", "--steps", "2", "--batch", "16")
    assert len(lines) == 1 and lines[0]["n_gpus"] == 1 and lines[0]["units"]["per_rank"] == [1]


def test_one_rank_launch_runs_the_exchange():
    """--launch: even --gpus 1 goes through torch.distributed.run, the process group and the exchange."""
    lines = _bench("--gpus", "1", "--launch", "--stub", "--workload", "r8", "--steps", "2", "--batch", "16")
    assert len(lines) == 1
    ln = lines[0]
    assert ln["n_gpus"] == 1 and ln["units"]["per_rank"] == [1]
    assert ln["exchange"]["backend"] == "gloo" and ln["exchange"]["ranks"] == 1
    assert ln["exchange"]["logits_rows_gathered"] == 1


@pytest.mark.gpu
def test_one_rank_nccl_exchange_on_device():
    """The NCCL communicator and the logits/counts exchange on the B200 (one rank: the box has one GPU)."""
    lines = _bench("--gpus", "1", "--launch", "--workload", "r8", "--steps", "2", "--warmup", "3",
                   "--no-cpu-baseline", "--no-autotune", timeout=900)
    assert len(lines) == 1, lines
    ln = lines[0]
    assert ln["exchange"]["backend"] == "nccl" and ln["exchange"]["ranks"] == 1
    assert ln["parity"]["status"] == "bit-exact", ln["parity"]


@pytest.mark.gpu
def test_two_ranks_share_one_gpu_device_path():
    """The multi-rank DEVICE path end to end on a one-GPU box: the launcher, two ranks each running its own
    range-batch through the CUDA-graph executor, the exchange (gloo here: NCCL needs one GPU per rank),
    the max-over-ranks timing, rank 0's logits bit-exact against the reference's."""
    lines = _bench("--gpus", "2", "--share-device", "--workload", "r8", "--steps", "2", "--warmup", "3",
                   "--no-cpu-baseline", "--no-autotune", timeout=900)
    assert len(lines) == 1, lines
    ln = lines[0]
    assert ln["n_gpus"] == 2 and ln["shared_device"] is True and ln["scaling"] == "weak"
    assert ln["units"] == {"kind": "range-batches", "per_rank": [1, 1], "total": 2, "covered_once": True}
    assert ln["parity"]["status"] == "bit-exact", ln["parity"]
    assert ln["value"] > 0 and ln["e2e"]["value"] > 0
