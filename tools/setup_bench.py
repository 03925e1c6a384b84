"""Setup time of a heterogeneous config-5-sized ensemble (every run its own
radial operator and coefficients: one eigenproblem, one phi1 matrix and one
Phi table per (run, component)): host `prepare` per operator set against the
batched on-device setup (`device_setup.prepare_device`).

    python tools/setup_bench.py [RUNS]      -> one JSON line
"""
import dataclasses
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs, integrators, operators as ops  # noqa: E402
from paper_2604_11558_b200.device_setup import prepare_device  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n1, n2 = 128, 256
base = configs.config5_member(0, (n1, n2))
bases = []
for j in range(R):
    rho = ops.build_lambda(n1, 1.0 + 0.5 * j / max(R - 1, 1), -1.95)      # domain-size sweep
    for c, f in zip(base.components, (1.0, 0.8 + 0.4 * j / max(R - 1, 1))):  # delta sweep
        bases.append(dataclasses.replace(c.ops, coeff=c.ops.coeff * f, rho=rho,
                                         rho_weights=ops.DiagonalWeights(rho.grid ** -(2.0 - 1.95))))
tau = 1e-3
torch.zeros(1, device="cuda")
prepare_device(bases[:4], tau)  # warm-up: library load, kernels
torch.cuda.synchronize()
t0 = time.perf_counter()
dev = prepare_device(bases, tau)
torch.cuda.synchronize()
t_dev = time.perf_counter() - t0
integrators._OP_CACHE.clear()
t0 = time.perf_counter()
host = [integrators.prepare(b, tau) for b in bases]
t_host = time.perf_counter() - t0
err = max(float(np.max(np.abs(d.phi1_rho - h.phi1_rho)) / np.max(np.abs(h.phi1_rho))) for d, h in zip(dev, host))
errm = max(float(np.max(np.abs(d.phi_mix.field - h.phi_mix.field))) for d, h in zip(dev, host))
print(json.dumps({"runs": R, "operator_sets": len(bases), "grid": [n1, n2], "distinct_eigenproblems": R,
                  "host_prepare_s": round(t_host, 3), "device_prepare_s": round(t_dev, 3),
                  "speedup": round(t_host / t_dev, 1), "phi1_rho_max_rel_diff": err, "phi_mix_max_abs_diff": errm,
                  "host_cores": len(os.sched_getaffinity(0))}))
