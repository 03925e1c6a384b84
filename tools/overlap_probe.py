"""Probe: does the HBM/smem-bound disk front overlap with the DMMA-bound
phi1_rho GEMM when the ensemble is split into two halves on two streams?
  python tools/overlap_probe.py base|serial|split|free [nsteps]
(set CURVIGPU_GEMM_CPS / CURVIGPU_FRONT_CPS to cap CTAs per SM)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.ensemble import ensemble_plan
from paper_2604_11558_b200.integrators import INT32_MAX

mode = sys.argv[1]
NS = int(sys.argv[2]) if len(sys.argv) > 2 else 200
R = 512
ens = configs.config5_inputs(0, R)
params = np.stack([[g, 0.1, 0.9] for g in ens.gammas])
W0 = torch.from_numpy(ens.states).cuda()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

if mode == "base":
    plan = ensemble_plan(ens.template, "schnakenberg", params, 1e-3, theta="fft")
    bad = torch.full((R, 2), INT32_MAX, dtype=torch.int32, device="cuda")
    s = W0.clone()
    plan.run(s, 0, 32, bad)
    torch.cuda.synchronize()
    ev0.record(); plan.run(s, 0, NS, bad); ev1.record(); torch.cuda.synchronize()
else:
    h = R // 2
    plans = [ensemble_plan(ens.template, "schnakenberg", params[k * h:(k + 1) * h], 1e-3, theta="fft") for k in (0, 1)]
    Ws = [W0[k * h:(k + 1) * h].clone() for k in (0, 1)]
    Os = [torch.empty_like(w) for w in Ws]
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    streams = [main, side] if mode != "serial" else [main, main]
    eF = [torch.cuda.Event(), torch.cuda.Event()]
    eG = [torch.cuda.Event(), torch.cuda.Event()]

    def step(first):
        for k in (0, 1):
            with torch.cuda.stream(streams[k]):
                if mode == "split":
                    if k == 1:
                        streams[1].wait_event(eF[0])
                    elif not first:
                        streams[0].wait_event(eF[1])
                plans[k].run_stage(-2, Ws[k], Os[k])
                eF[k].record()
        for k in (0, 1):
            with torch.cuda.stream(streams[k]):
                if mode == "split":
                    if k == 1:
                        streams[1].wait_event(eG[0])
                    elif not first:
                        streams[0].wait_event(eG[1])
                plans[k].run_stage(1, Ws[k], Os[k])
                eG[k].record()
        for k in (0, 1):
            Ws[k], Os[k] = Os[k], Ws[k]

    for t in range(8):
        step(t == 0)
    torch.cuda.synchronize()
    ev0.record()
    for t in range(NS):
        step(False)
    main.wait_stream(side)
    ev1.record()
    torch.cuda.synchronize()
ms = ev0.elapsed_time(ev1) / NS
print(json.dumps({"mode": mode, "gemm_cps": os.environ.get("CURVIGPU_GEMM_CPS"),
                  "front_cps": os.environ.get("CURVIGPU_FRONT_CPS"), "ms_per_step": round(ms, 4)}))
