"""Graph-timed kernels of one step (50 launches per graph, CUDA events) for
BASELINE configs 1-5 at full size: CONFIGS=1,2,3,4 THETAS=fft,gemm."""
import json, os, sys
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import numpy as np
import torch
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.ensemble import ensemble_plan
from paper_2604_11558_b200.integrators import SplitPlan, prepare
from small_gemm_sweep import graph_time  # noqa: E402

PEAK = 37.05
for k in [int(x) for x in os.environ.get("CONFIGS", "1,2,3,4").split(",")]:
    for theta in os.environ.get("THETAS", "fft").split(","):
        if k == 5:  # the bench workload: 512-run config-5 ensemble
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
        o = torch.empty_like(W)
        rows = []
        for st in plan.step_kernels():
            fl, by = plan.stage_info(st)
            us = graph_time(lambda: plan.run_stage(st, W, o))
            rows.append({"k": st, "us": round(us, 2), "tflops": round(fl / us / 1e6, 2) if fl else None,
                         "frac": round(fl / us / 1e6 / PEAK, 3) if fl else None,
                         "gbs": round(by / us / 1e3, 1) if (by and not fl) else None})
        print(json.dumps({"config": k, "theta": theta, "kernels": rows}), flush=True)
        plan.close()
