"""Run each kernel of one config-5 step once (after a warm-up step) so an
ncu capture sees exactly one launch per kernel, in step order.  Also writes
the kernel-name order to gpurun_out/step_kernels_<theta>.json."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.ensemble import ensemble_plan
from paper_2604_11558_b200.integrators import INT32_MAX

theta = os.environ.get("THETA", "fft")
ens = configs.config5_inputs(0, 512)
params = np.stack([[g, 0.1, 0.9] for g in ens.gammas])
plan = ensemble_plan(ens.template, "schnakenberg", params, 1e-3, theta=theta)
W = torch.from_numpy(ens.states).cuda()
out = torch.empty_like(W)
bad = torch.full((512, 2), INT32_MAX, dtype=torch.int32, device="cuda")
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
json.dump(names, open(f"gpurun_out/step_kernels_{theta}.json", "w"))
print("kernels", names)
