"""Host logic of the ensemble path on CPU: shard ranges and the rank-0
gather, exercised with a real world_size-2 gloo process group."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_11558_b200.ensemble import gather_fields, shard_range


@pytest.mark.parametrize("total,world", [(512, 1), (512, 2), (512, 8), (7, 3), (3, 8)])
def test_shards_partition_the_runs(total, world):
    covered = []
    for r in range(world):
        lo, hi = shard_range(total, r, world)
        assert 0 <= lo <= hi <= total
        covered.extend(range(lo, hi))
    assert covered == list(range(total))
    sizes = [shard_range(total, r, world)[1] - shard_range(total, r, world)[0] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def test_bad_rank_rejected():
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(total, rank, world)
    local = torch.arange(lo, hi, dtype=torch.float64).view(-1, 1, 1, 1).repeat(1, 2, 3, 4)
    local[:, 1] *= -1
    out = gather_fields(local, total)
    if rank == 0:
        q.put(out.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [7, 8])
def test_gather_to_rank0_world2_gloo(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got.shape == (total, 2, 3, 4)
    for i in range(total):
        assert (got[i, 0] == i).all() and (got[i, 1] == -i).all()
