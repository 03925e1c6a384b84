"""Per-GPU config-5 throughput (THETA=fft default) at the shard sizes of an N-GPU run (512 / N
runs per rank, N = 1, 2, 4, 8) on one GPU, lanes 1..4: what the scaling run's
per-rank step costs.  CUDA-event timed plan.run over 200 time steps."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.ensemble import ensemble_plan

STEPS = 200
for n in (1, 2, 4, 8):
    runs = 512 // n
    ens = configs.config5_inputs(0, runs)
    params = np.stack([[g, 0.1, 0.9] for g in ens.gammas])
    for lanes in (None, 1, 2, 3, 4):
        if lanes is None:
            os.environ.pop("CURVIGPU_LANES", None)
        else:
            os.environ["CURVIGPU_LANES"] = str(lanes)
        plan = ensemble_plan(ens.template, "schnakenberg", params, 1e-3, theta=os.environ.get("THETA", "fft"))
        W0 = torch.from_numpy(ens.states).cuda()
        bad = torch.full((runs, 2), 2**31 - 1, dtype=torch.int32, device="cuda")
        s = W0.clone()
        plan.run(s, 0, 32, bad)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.copy_(W0)
        e0.record()
        plan.run(s, 0, STEPS, bad)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / STEPS
        dof = runs * 2 * 128 * 256
        print(json.dumps({"gpus_emulated": n, "runs": runs, "lanes": lanes or f"default({plan.lanes})",
                          "us_per_step": round(us, 2), "dof_steps_per_s": dof / us * 1e6,
                          "us_per_run_step": round(us / runs, 4)}), flush=True)
        plan.close()
