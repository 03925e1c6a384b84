"""Per-stage determinism: each kernel of one full-size step (CONFIG, THETA)
run REPS times on the same input; reports differing entries per stage and,
for GEMM stages, which tiles / warp regions differ (64x64 tiles, 32x32 warps)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.integrators import SplitPlan, prepare

k = int(os.environ.get("CONFIG", "4"))
reps = int(os.environ.get("REPS", "30"))
theta = os.environ.get("THETA", "gemm")
system = configs.BUILDERS[k]()
m, ts = configs.STEPS[k]
geos = [prepare(c.ops, ts / m) for c in system.components]
plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :], theta=theta)
W = torch.from_numpy(np.stack([c.initial for c in system.components])[None].copy()).cuda()
out = torch.empty_like(W)
kernels = plan.step_kernels()
# fill the workspaces with one real step so every stage sees realistic inputs
for st in kernels:
    plan.run_stage(st, W, out)
torch.cuda.synchronize()
sel = [int(x) for x in os.environ['STAGE'].split(',')] if 'STAGE' in os.environ else kernels
for st in sel:
    res = []
    for r in range(reps):
        plan.run_stage(st, W, out)
        torch.cuda.synchronize()
        # output of stage st: last stage -> out, else its dst workspace
        ws = [plan.workspace(0).clone(), plan.workspace(1).clone(), out.clone()]
        res.append(ws)
    nd = [sum(int((a != b).sum()) for a, b in zip(res[0], x)) for x in res[1:]]
    print(os.environ.get("CURVIGPU_LIB", "default lib").split("/")[-1], "stage", st, "reps", reps,
          "bad reps", sum(1 for v in nd if v), "ndiff", sorted(set(nd)), flush=True)
    if any(nd):
        r = next(i for i, v in enumerate(nd) if v) + 1
        for wi in range(3):
            d = (res[0][wi] != res[r][wi])
            if d.any():
                idx = torch.nonzero(d.reshape(d.shape[0] * d.shape[1], -1) if False else d)[:10]
                print("   buffer", wi, "shape", tuple(d.shape), "first diffs", idx.tolist()[:5],
                      "count", int(d.sum()), flush=True)
