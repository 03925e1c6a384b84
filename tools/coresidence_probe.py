"""Probe: can the fused disk front and the phi1_rho GEMM run concurrently on
the same SMs?  Times F alone, G alone and F || G on two streams (20 reps).
Run with CURVIGPU_GEMM_CPS=1 CURVIGPU_FRONT_CPS=1 (one CTA of each per SM)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.ensemble import ensemble_plan

R = 256
ens = configs.config5_inputs(0, R)
params = np.stack([[g, 0.1, 0.9] for g in ens.gammas])
pa = ensemble_plan(ens.template, "schnakenberg", params, 1e-3, theta="fft")
pb = ensemble_plan(ens.template, "schnakenberg", params, 1e-3, theta="fft")
W = torch.from_numpy(ens.states).cuda()
Oa, Ob = torch.empty_like(W), torch.empty_like(W)
side = torch.cuda.Stream()
main = torch.cuda.current_stream()
REPS = 20


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    side_done = torch.cuda.Event()
    side_done.record(side)
    main.wait_event(side_done)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / REPS


def F():
    for _ in range(REPS):
        pa.run_stage(-2, W, Oa)


def G():
    for _ in range(REPS):
        pb.run_stage(1, W, Ob)


def both():
    ev = torch.cuda.Event()
    ev.record()
    side.wait_event(ev)
    with torch.cuda.stream(side):
        G()
    F()


def interleaved():
    ev = torch.cuda.Event()
    ev.record()
    side.wait_event(ev)
    for _ in range(REPS):
        pa.run_stage(-2, W, Oa)
        with torch.cuda.stream(side):
            pb.run_stage(1, W, Ob)


print(json.dumps({"gemm_cps": os.environ.get("CURVIGPU_GEMM_CPS"), "front_cps": os.environ.get("CURVIGPU_FRONT_CPS"),
                  "F_ms": round(timed(F), 4), "G_ms": round(timed(G), 4), "F||G_ms": round(timed(both), 4),
                  "interleaved_ms": round(timed(interleaved), 4)}))
