"""Determinism stress: full-size ball, REPS reruns of NSTEP graph-replayed
steps from the same state; prints how many distinct results appear."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.integrators import INT32_MAX, SplitPlan, prepare

reps = int(os.environ.get("REPS", "12"))
nstep = int(os.environ.get("NSTEP", "40"))
theta = os.environ.get("THETA", "gemm")
system = configs.config4()
geos = [prepare(c.ops, 1e-2) for c in system.components]
plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :], theta=theta)
W = torch.from_numpy(np.stack([c.initial for c in system.components])[None].copy()).cuda()
bad = torch.full((1, 2), INT32_MAX, dtype=torch.int32, device="cuda")
finals = []
for rep in range(reps):
    s = W.clone()
    plan.run(s, 0, nstep, bad)
    torch.cuda.synchronize()
    finals.append(s.cpu())
distinct = []
for f in finals:
    if not any(torch.equal(f, d) for d in distinct):
        distinct.append(f)
diffs = [int((f != finals[0]).sum()) for f in finals]
print({k: os.environ.get(k) for k in ("CURVIGPU_MAX_CARVEOUT", "CURVIGPU_GEMM_CPS", "CURVIGPU_NOPERSIST")},
      "reps", reps, "distinct", len(distinct), "ndiff_vs_first", diffs, flush=True)
