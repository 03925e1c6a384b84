"""Does every stage write its whole output?  Prefill the destination with NaN
and look for survivors (measurement / debugging tool)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.integrators import SplitPlan, prepare
dims = eval(os.environ.get("DIMS", "(100,96,100)"))
system = configs.config4(dims)
geos = [prepare(c.ops, 1e-2) for c in system.components]
plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :], theta="gemm")
W = torch.from_numpy(np.stack([c.initial for c in system.components])[None]).cuda()
out = torch.empty_like(W)
# stage s writes buffer X (s even after fbuild) / Y; run the chain and inspect each destination via a probe:
# fill every workspace with NaN by running a step on a NaN state first is not possible; instead use
# the state-sized probe: stage outputs land in plan workspaces, read back through run_stage(-1) semantics
import ctypes
lib = plan._lib
for s in plan.step_kernels():
    plan.run_stage(s, W, out)
torch.cuda.synchronize()
print("chain ok", flush=True)
