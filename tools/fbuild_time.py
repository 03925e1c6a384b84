"""Graph-timed F-build kernel (stage -1) of configs 3 and 4 (50 launches per graph)."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.integrators import SplitPlan, prepare
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
from small_gemm_sweep import graph_time  # noqa: E402

out = {}
for k in (3, 4):
    system = configs.BUILDERS[k]()
    m, ts = configs.STEPS[k]
    geos = [prepare(c.ops, ts / m) for c in system.components]
    plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :], theta="fft")
    W = torch.from_numpy(np.stack([c.initial for c in system.components])[None].copy()).cuda()
    o = torch.empty_like(W)
    out[f"c{k}_fbuild_us"] = round(graph_time(lambda: plan.run_stage(-1, W, o)), 2)
print(os.environ.get("CURVIGPU_LIB", "default"), json.dumps(out))
