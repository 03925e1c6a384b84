"""Run each kernel of one step once (after a warm-up step) so an ncu capture
sees exactly one launch per kernel, in step order.  CONFIG=5 (default):
the config-5 ensemble; CONFIG=1..4: that BASELINE config at full size.
Writes the kernel-name order to gpurun_out/step_kernels_<theta>[_c<k>].json."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.ensemble import ensemble_plan
from paper_2604_11558_b200.integrators import INT32_MAX, SplitPlan, prepare

theta = os.environ.get("THETA", "fft")
k = int(os.environ.get("CONFIG", "5"))
if k == 5:
    ens = configs.config5_inputs(0, 512)
    params = np.stack([[g, 0.1, 0.9] for g in ens.gammas])
    plan = ensemble_plan(ens.template, "schnakenberg", params, 1e-3, theta=theta)
    W = torch.from_numpy(ens.states).cuda()
else:
    system = configs.BUILDERS[k]()
    m, ts = configs.STEPS[k]
    geos = [prepare(c.ops, ts / m) for c in system.components]
    plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :], theta=theta)
    W = torch.from_numpy(np.stack([c.initial for c in system.components])[None].copy()).cuda()
out = torch.empty_like(W)
bad = torch.full(tuple(W.shape[:2]), INT32_MAX, dtype=torch.int32, device="cuda")
s = W.clone()
plan.run(s, 0, 1, bad)  # warm-up step (not profiled: -s skips it)
torch.cuda.synchronize()
names = []
for st in plan.step_kernels():
    fl, by = plan.stage_info(st)
    names.append({-1: "fbuild", -2: "fused_fbuild_theta_fft"}.get(st, f"gemm_stage{st}" if fl else f"theta_fft_stage{st}"))
    plan.run_stage(st, W, out)
torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(names, open(f"gpurun_out/step_kernels_{theta}{'' if k == 5 else f'_c{k}'}.json", "w"))
print("kernels", names)
