"""Probe: config-5 ensemble split into L independent lanes (sub-plans on their
own streams, graph-replayed cg_run chunks), ms per time step.
  python tools/lanes_probe.py L [nsteps]"""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.ensemble import ensemble_plan
from paper_2604_11558_b200.integrators import INT32_MAX

L = int(sys.argv[1])
NS = int(sys.argv[2]) if len(sys.argv) > 2 else 200
R = 512
ens = configs.config5_inputs(0, R)
params = np.stack([[g, 0.1, 0.9] for g in ens.gammas])
W0 = torch.from_numpy(ens.states).cuda()
cuts = [R * k // L for k in range(L + 1)]
plans = [ensemble_plan(ens.template, "schnakenberg", params[cuts[k]:cuts[k + 1]], 1e-3, theta="fft") for k in range(L)]
Ws = [W0[cuts[k]:cuts[k + 1]].clone() for k in range(L)]
bads = [torch.full((cuts[k + 1] - cuts[k], 2), INT32_MAX, dtype=torch.int32, device="cuda") for k in range(L)]
main = torch.cuda.current_stream()
streams = [main] + [torch.cuda.Stream() for _ in range(L - 1)]


def run(n):
    ev = torch.cuda.Event()
    ev.record(main)
    for k in range(L):
        streams[k].wait_event(ev)
        with torch.cuda.stream(streams[k]):
            plans[k].run(Ws[k], 0, n, bads[k])
    for k in range(1, L):
        main.wait_stream(streams[k])


run(32)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(main)
run(NS)
e1.record(main)
torch.cuda.synchronize()
print(json.dumps({"lanes": L, "ms_per_step": round(e0.elapsed_time(e1) / NS, 4)}))
