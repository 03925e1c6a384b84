import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.integrators import INT32_MAX, SplitPlan, prepare

dims = eval(os.environ.get("DIMS", "None"))
system = configs.config4(dims)
geos = [prepare(c.ops, 1e-2) for c in system.components]
plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :], theta="gemm")
W = torch.from_numpy(np.stack([c.initial for c in system.components])[None]).cuda()
bad = torch.full((1, 2), INT32_MAX, dtype=torch.int32, device="cuda")
finals = []
for rep in range(8):
    s = W.clone()
    if os.environ.get("EAGER"):
        for k in range(40):
            plan.run(s, k, 1, bad)
            if os.environ.get("SYNC"):
                torch.cuda.synchronize()
    else:
        plan.run(s, 0, 40, bad)
    torch.cuda.synchronize()
    finals.append(s.clone())
print(os.environ.get("DIMS"), os.environ.get("EAGER"), os.environ.get("SYNC"), os.environ.get("CUDA_LAUNCH_BLOCKING"),
      "deterministic:", all(torch.equal(finals[0], f) for f in finals[1:]),
      "maxdiff:", max(float((finals[0] - f).abs().max()) for f in finals[1:]), flush=True)
