"""GPU per-config step times (bench.per_config_gpu) plus per-kernel times of
one step, configs 1-4 at full size, both theta modes.  Measurement tool."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import bench
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.integrators import SplitPlan, prepare

for k in (1, 2, 3, 4):
    for t in ("fft", "gemm"):
        r = bench.per_config_gpu(k, theta=t)
        system = configs.BUILDERS[k]()
        m, ts = configs.STEPS[k]
        geos = [prepare(c.ops, ts / m) for c in system.components]
        plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :], theta=t)
        W = torch.from_numpy(np.stack([c.initial for c in system.components])[None].copy()).cuda()
        out = torch.empty_like(W)
        ks = []
        for st in plan.step_kernels():
            for _ in range(3):
                plan.run_stage(st, W, out)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                plan.run_stage(st, W, out)
            e1.record()
            e1.synchronize()
            fl, by = plan.stage_info(st)
            us = e0.elapsed_time(e1) / 20 * 1e3
            ks.append({"k": st, "us": round(us, 2), "tflops": round(fl / us / 1e6, 2) if fl else None})
        print(json.dumps({"config": k, "theta": t, "ms_per_step": round(r["ms_per_step"], 4),
                          "gemm_frac": round(r["gemm_chain_frac_fp64_peak"], 3), "kernels": ks}), flush=True)
