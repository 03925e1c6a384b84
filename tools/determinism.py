"""Bitwise determinism of every kernel of one step (cg_run_stage repeated on
identical inputs) and of whole runs; localises races.  Run under gpurun."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.integrators import INT32_MAX, SplitPlan, prepare


def check(k, theta, reps=30):
    system = configs.BUILDERS[k]()
    m, ts = configs.STEPS[k]
    geos = [prepare(c.ops, ts / m) for c in system.components]
    plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :], theta=theta)
    W = torch.from_numpy(np.stack([c.initial for c in system.components])[None]).cuda()
    # prime the workspaces with one full step so every stage sees realistic inputs
    st = W.clone()
    bad = torch.full((1, 2), INT32_MAX, dtype=torch.int32, device="cuda")
    plan.run(st, 0, 1, bad)
    for stage in plan.step_kernels():
        outs = []
        for _ in range(reps):
            out = torch.zeros_like(W)
            plan.run_stage(stage, W, out)
            torch.cuda.synchronize()
            outs.append(out.clone())
        same = all(torch.equal(outs[0], o) for o in outs[1:])
        print(f"config {k} theta {theta} stage {stage}: deterministic={same}", flush=True)
    finals = []
    for _ in range(6):
        s = W.clone()
        plan.run(s, 0, 40, bad)
        torch.cuda.synchronize()
        finals.append(s.clone())
    print(f"config {k} theta {theta} run40 deterministic={all(torch.equal(finals[0], f) for f in finals[1:])}", flush=True)


for k in (4, 3, 2, 1):
    for theta in ("gemm", "fft"):
        check(k, theta)
