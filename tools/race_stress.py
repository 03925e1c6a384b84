"""Race detection by rerun statistics (compute-sanitizer is closed on the GPU
pool): every kernel of one step of every BASELINE config, in both theta
formulations and every GEMM tile configuration that the plan would accept,
is rerun REPS times on fixed inputs (cg_run_stage) and its output compared
bitwise with the first run.  A shared-memory or proxy race shows up as a
run-to-run difference (the r01 stage-ring WAR race appeared in ~1/200 runs).

    python tools/race_stress.py [REPS]      -> one JSON line per (config, theta, cfg, stage)
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs  # noqa: E402
from paper_2604_11558_b200.ensemble import ensemble_plan  # noqa: E402
from paper_2604_11558_b200.integrators import SplitPlan, prepare  # noqa: E402

REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 100


def plan_for(k, theta):
    if k == 5:
        ens = configs.config5_inputs(0, 64)
        params = np.stack([[g, 0.1, 0.9] for g in ens.gammas])
        plan = ensemble_plan(ens.template, "schnakenberg", params, 1e-3, theta=theta)
        return plan, torch.from_numpy(ens.states).cuda()
    system = configs.BUILDERS[k]()
    m, ts = configs.STEPS[k]
    geos = [prepare(c.ops, ts / m) for c in system.components]
    plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :], theta=theta)
    return plan, torch.from_numpy(np.stack([c.initial for c in system.components])[None].copy()).cuda()


def stage_output(plan, st, W, out):
    plan.run_stage(st, W, out)
    if st >= 0 and st == plan.stage_count() - 1:
        return out.clone()
    # intermediate stages write the plan's workspaces: read the one they produced
    return torch.cat([plan.workspace(0).flatten(), plan.workspace(1).flatten()])


def main():
    os.environ["CURVIGPU_LANES"] = "1"
    cfgs = (None, "resident", "2", "7", "8", "9", "11", "12", "13", "15", "18", "19")
    if os.environ.get("RS_CFGS"):  # e.g. RS_CFGS=default,12,18 RS_CONFIGS=4
        cfgs = tuple(None if c == "default" else c for c in os.environ["RS_CFGS"].split(","))
    ks = tuple(int(c) for c in os.environ.get("RS_CONFIGS", "1,2,3,4,5").split(","))
    for cfg in cfgs:
        os.environ.pop("CURVIGPU_TILE_CFG", None)
        os.environ.pop("CURVIGPU_RESIDENT", None)
        if cfg == "resident":  # every eligible stage through the resident-operator kernel
            os.environ["CURVIGPU_RESIDENT"] = "1"
        elif cfg:
            os.environ["CURVIGPU_TILE_CFG"] = cfg
        for k in ks:
            for theta in ("fft", "gemm"):
                if cfg and cfg != "resident" and k == 5:
                    continue
                plan, W = plan_for(k, theta)
                out = torch.empty_like(W)
                kernels = plan.step_kernels()
                for st in kernels:  # fill the workspaces in step order once
                    plan.run_stage(st, W, out)
                for st in kernels:
                    # inputs of stage st are the workspaces left by the step order: re-run the
                    # prefix so every rerun of st sees identical inputs
                    first, ndiff = None, 0
                    for _ in range(REPS):
                        for pre in kernels[: kernels.index(st)]:
                            plan.run_stage(pre, W, out)
                        got = stage_output(plan, st, W, out)
                        if first is None:
                            first = got
                        elif not torch.equal(torch.nan_to_num(got, nan=7.0), torch.nan_to_num(first, nan=7.0)):
                            ndiff += 1
                    print(json.dumps({"config": k, "theta": theta, "tile_cfg": cfg or "default", "stage": st,
                                      "reps": REPS, "runs_differing": ndiff}), flush=True)
                plan.close()


def cluster_runs():
    """The cluster step kernel (all steps of cg_run in one launch, DSMEM hand-over
    on tx-count mbarriers): REPS reruns of 60 steps from the same state."""
    os.environ.pop("CURVIGPU_TILE_CFG", None)
    os.environ.pop("CURVIGPU_RESIDENT", None)
    for dims in ((64, 128), (32, 64)):
        system = configs.BUILDERS[1](dims)
        geos = [prepare(c.ops, 1e-3) for c in system.components]
        plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :], theta="fft")
        W0 = torch.from_numpy(np.stack([c.initial for c in system.components])[None].copy()).cuda()
        bad = torch.full((1, 2), 2**31 - 1, dtype=torch.int32, device="cuda")
        first, ndiff = None, 0
        for _ in range(REPS):
            state = W0.clone()
            plan.run(state, 0, 60, bad)
            if first is None:
                first = state.clone()
            elif not torch.equal(state, first):
                ndiff += 1
        print(json.dumps({"config": 1, "dims": list(dims), "kernel": "disk_cluster_kernel", "steps": 60,
                          "reps": REPS, "runs_differing": ndiff}), flush=True)
        plan.close()


if __name__ == "__main__":
    main()
    if not os.environ.get("RS_CFGS"):
        cluster_runs()
