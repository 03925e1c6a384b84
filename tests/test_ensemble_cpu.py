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


def _agree_worker(rank, world, port, q):
    from paper_2604_11558_b200.ensemble import agree

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q.put((rank, agree(10 + 5 * rank, "min"), agree(10 + 5 * rank, "max")))
    dist.barrier()
    dist.destroy_process_group()


def test_ranks_agree_on_min_and_max_world2_gloo():
    """The all-reduce run_ensemble uses so that a divergence or setup error
    on one shard is raised by every rank before the gather."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got == [(0, 10, 15), (1, 10, 15)]


def test_agree_without_process_group_is_identity():
    from paper_2604_11558_b200.ensemble import agree

    assert agree(7, "min") == 7 and agree(-3, "max") == -3


def test_bench_refuses_more_gpus_than_visible():
    """bench.py --gpus N without a launcher re-execs under torchrun, and
    refuses loudly when fewer than N devices are visible (no silent 1-rank run)."""
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2
    assert "needs 2 visible CUDA devices" in r.stderr


def test_bench_refuses_world_size_mismatch():
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0", CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0
    assert "launcher started 1 rank" in r.stderr
