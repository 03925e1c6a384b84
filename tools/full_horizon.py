"""BASELINE configs 1-4 over their FULL horizons (configs.STEPS) at full size:
the CUDA path (run_simulation -> cg_run) against the CPU oracle on the same
initial data; relative inf-norm per component and wall time of both.
    CONFIGS=1,2,3,4 python tools/full_horizon.py > gpurun_out/full_horizon.jsonl"""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from oracle import configs as ocfg
from oracle import curvi_oracle as orc
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.integrators import run_simulation

for k in [int(x) for x in os.environ.get("CONFIGS", "1,2,3,4").split(",")]:
    m, t_star = configs.STEPS[k]
    m = int(os.environ.get("STEPS", m))
    t_star = t_star * m / configs.STEPS[k][0]
    system = configs.BUILDERS[k]()
    run_simulation(system, 2, 2 * t_star / m)  # plan creation / module load outside the timing
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = run_simulation(system, m, t_star)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    osys = ocfg.BUILDERS[k](initial=[c.initial for c in system.components])
    t0 = time.perf_counter()
    ref = orc.physical(osys, orc.integrate(osys, m, t_star))
    cpu_s = time.perf_counter() - t0
    errs = {}
    for c in system.components:
        got = res.fields[c.name] + c.lift
        errs[c.name] = float(np.max(np.abs(got - ref[c.name])) / np.max(np.abs(ref[c.name])))
    print(json.dumps({"config": configs.NAMES[k], "steps": m, "t_star": t_star, "rel_inf": errs,
                      "gpu_run_s": round(gpu_s, 3), "oracle_cpu_s": round(cpu_s, 1),
                      "cpu_threads": os.cpu_count()}), flush=True)

if os.environ.get("ENSEMBLE", "1") != "0":
    # config 5: the whole 512-run ensemble over its full horizon on the GPU, every
    # EVERY-th member (and the last) against the oracle
    from paper_2604_11558_b200.ensemble import ensemble_plan

    every = int(os.environ.get("EVERY", "16"))
    m, t_star = configs.STEPS[5]
    ens = configs.config5_inputs(0, configs.ENSEMBLE_RUNS)
    params = np.stack([[g, 0.1, 0.9] for g in ens.gammas])
    plan = ensemble_plan(ens.template, "schnakenberg", params, t_star / m)
    state = torch.from_numpy(ens.states).cuda()
    bad = torch.full((configs.ENSEMBLE_RUNS, 2), 2**31 - 1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.run(state, 0, m, bad)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    out = state.cpu().numpy()
    picks = sorted(set(range(0, configs.ENSEMBLE_RUNS, every)) | {configs.ENSEMBLE_RUNS - 1})
    worst, t0 = 0.0, time.perf_counter()
    for i in picks:
        osys = ocfg.config5_member(i, initial=[ens.states[i, 0], ens.states[i, 1]])
        ref = orc.physical(osys, orc.integrate(osys, m, t_star))
        for c, (name, lift) in enumerate((("u", 1.0), ("v", 0.9))):
            worst = max(worst, float(np.max(np.abs(out[i, c] + lift - ref[name])) / np.max(np.abs(ref[name]))))
    print(json.dumps({"config": "disk_schnakenberg_ensemble_512x128x256", "steps": m, "t_star": t_star,
                      "members_checked": len(picks), "worst_rel_inf": worst, "diverged": int((bad.cpu().numpy() < 2**31 - 1).any(axis=1).sum()),
                      "gpu_run_s_all_512": round(gpu_s, 3), "oracle_cpu_s_checked_members": round(time.perf_counter() - t0, 1),
                      "cpu_threads": os.cpu_count()}), flush=True)
