"""The sharded ensemble path with real ranks on the GPU.

Two processes share cuda:0 over a gloo group (the pool leases one GPU per
call; gather_fields stages the device blocks through host memory for gloo).
The ranks' kernels never wait on each other -- shards are independent runs
and the only exchange is the final gather -- so this is the multi-rank code
path itself, not a stand-in for a collective kernel.  The NCCL variant runs
when the box has two or more GPUs.

Checks: the gathered fields equal the single-process run bitwise; a member
that diverges in ONE shard makes every rank raise the same DivergenceError
(no rank is left blocked in the gather); a setup error on one
rank is raised on all of them.
"""

import dataclasses
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = (16, 32)
MEMBERS = list(range(40, 47))  # 7 runs: ranks get 3 and 4
STEPS, T_STAR = 20, 0.02


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _members(mode):
    from paper_2604_11558_b200 import configs as pcfg
    from paper_2604_11558_b200.models import Kinetics

    ms = [pcfg.config5_member(i, DIMS) for i in MEMBERS]
    if mode == "diverge":  # one member of rank 1's shard blows up
        s = ms[5]
        ms[5] = dataclasses.replace(s, kinetics=Kinetics("schnakenberg", {"gamma": 5e8, "a": 0.1, "b": 0.9}))
    if mode == "badsetup":  # rank 1's shard has a member with a foreign component list
        s = ms[4]
        ms[4] = dataclasses.replace(s, components=list(reversed(s.components)))
    return ms


def _worker(rank, world, port, backend, mode, q):
    import torch
    import torch.distributed as dist

    from paper_2604_11558_b200.ensemble import run_ensemble
    from paper_2604_11558_b200.integrators import DivergenceError

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    kw = {"device_id": torch.device("cuda", dev)} if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    try:
        res = run_ensemble(_members(mode), STEPS, T_STAR, raise_on_divergence=(mode == "diverge"))
        q.put((rank, "ok", res.fields if rank == 0 else None, res.first_bad, res.start, res.stop))
    except DivergenceError as e:
        q.put((rank, "diverged", e.step, None, None, None))
    except Exception as e:  # noqa: BLE001 -- reported to the parent
        q.put((rank, "error", f"{type(e).__name__}: {e}", None, None, None))
    dist.barrier()
    dist.destroy_process_group()


def _run(backend, mode, world=2):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        item = q.get(timeout=300)
        out[item[0]] = item[1:]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


def _single(mode):
    from paper_2604_11558_b200.ensemble import run_ensemble

    return run_ensemble(_members(mode), STEPS, T_STAR)


def _backends():
    import torch

    out = ["gloo"]
    if torch.cuda.device_count() >= 2:
        out.append("nccl")
    return out


@pytest.mark.parametrize("backend", _backends())
def test_two_ranks_gather_equals_single_process_bitwise(backend):
    got = _run(backend, "plain")
    ref = _single("plain")
    assert got[0][0] == "ok" and got[1][0] == "ok"
    assert (got[0][3], got[0][4]) == (0, 3) and (got[1][3], got[1][4]) == (3, 7)
    assert got[0][1].shape == ref.fields.shape
    assert np.array_equal(got[0][1], ref.fields)
    assert got[1][1] is None
    assert np.array_equal(np.concatenate([got[0][2], got[1][2]]), ref.first_bad)


@pytest.mark.parametrize("backend", _backends())
def test_divergence_in_one_shard_is_raised_by_every_rank(backend):
    got = _run(backend, "diverge")
    ref = _single("diverge")
    want = int(ref.first_bad.min())
    assert want < 2**31 - 1
    assert got[0] == ("diverged", want, None, None, None)
    assert got[1] == ("diverged", want, None, None, None)


def test_setup_error_in_one_shard_is_raised_by_every_rank():
    got = _run("gloo", "badsetup")
    assert got[0][0] == "error" and "rank 1" in got[0][1]
    assert got[1][0] == "error" and "NotImplementedError" in got[1][1]


def test_single_rank_nccl_group_takes_the_collective_path():
    """The pool leases one GPU, so the NCCL code path (device-side `agree`
    all-reduce, `gather_fields` over NCCL) is exercised with a world of one:
    same result as the run without a process group, bitwise."""
    got = _run("nccl", "plain", world=1)
    ref = _single("plain")
    assert got[0][0] == "ok" and (got[0][3], got[0][4]) == (0, len(MEMBERS))
    assert np.array_equal(got[0][1], ref.fields)
    assert np.array_equal(got[0][2], ref.first_bad)
