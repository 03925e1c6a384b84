#!/usr/bin/env python
"""Time every GEMM stage of every BASELINE config under each tile config
(CURVIGPU_TILE_CFG override) with CUDA events; prints one JSON line per
(config, stage, tile cfg).  Measurement tool, run under gpurun."""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_11558_b200 import configs  # noqa: E402
from paper_2604_11558_b200.integrators import SplitPlan, prepare  # noqa: E402

PEAK = 37.05


def plan_for(k, runs=None):
    if k == 5:
        ens = configs.config5_inputs(0, runs or 512)
        geos = [prepare(c.ops, 1e-3) for c in ens.template.components]
        params = np.stack([[g, 0.1, 0.9] for g in ens.gammas])
        return SplitPlan(geos, len(ens.gammas), "schnakenberg", params, lifts=[1.0, 0.9]), ens.states
    system = configs.BUILDERS[k]()
    m, ts = configs.STEPS[k]
    geos = [prepare(c.ops, ts / m) for c in system.components]
    plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :])
    return plan, np.stack([c.initial for c in system.components])[None]


def time_stage(plan, stage, W, out, reps=20):
    for _ in range(3):
        plan.run_stage(stage, W, out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        plan.run_stage(stage, W, out)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    cfgs = [int(x) for x in os.environ.get("SWEEP_CFGS", "0,1,2,3,4,5,6").split(",")]
    which = [int(x) for x in os.environ.get("SWEEP_CONFIGS", "5,1,2,3,4").split(",")]
    for k in which:
        for cfg in cfgs:
            os.environ["CURVIGPU_TILE_CFG"] = str(cfg)
            plan, host = plan_for(k)
            W = torch.from_numpy(np.ascontiguousarray(host)).cuda()
            out = torch.empty_like(W)
            for st in range(-1, plan.stage_count()):
                ms = time_stage(plan, st, W, out)
                fl, by = plan.stage_info(st)
                rec = {"config": k, "cfg": cfg, "stage": st, "ms": round(ms, 4)}
                if fl:
                    rec["tflops"] = round(fl / ms / 1e9, 2)
                    rec["frac"] = round(fl / ms / 1e9 / PEAK, 3)
                else:
                    rec["gbs"] = round(by / ms / 1e6, 1)
                print(json.dumps(rec), flush=True)
            plan.close()
            del W, out
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
