import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.integrators import INT32_MAX, SplitPlan, prepare
dims = eval(os.environ.get("DIMS", "(100,96,100)"))
stage = int(os.environ.get("STAGE", "2"))
system = configs.config4(dims)
geos = [prepare(c.ops, 1e-2) for c in system.components]
plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :], theta="gemm")
W = torch.from_numpy(np.stack([c.initial for c in system.components])[None]).cuda()
out = torch.empty_like(W)
for s in plan.step_kernels():
    plan.run_stage(s, W, out)
    if s == stage:
        break
torch.cuda.synchronize()
print("done", flush=True)
