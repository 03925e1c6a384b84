"""Small-shape workload for compute-sanitizer (racecheck / synccheck /
memcheck): every kernel family of libcurvigpu at shapes that finish in
seconds under instrumentation.

    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize.py
    compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize.py

Covers: the F-build (all geometries), both theta formulations (DMMA GEMM pair
and the FFT propagator), every GEMM tile configuration incl. the 2- and
4-CTA split-K clusters (CURVIGPU_TILE_CFG), the ball's chained polar-mode
kernel (both chain tiles) and its unchained form, the fused disk front in
its three CTA shapes, lanes, the partial-tile TMA-store path (odd / n=100
extents), the coupled bulk-surface step and the diagnostics reductions.
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch

    from paper_2604_11558_b200 import configs as pcfg
    from paper_2604_11558_b200 import integrators, models
    from paper_2604_11558_b200.ensemble import run_ensemble
    from paper_2604_11558_b200.integrators import run_simulation

    quick = "--quick" in sys.argv
    t0 = time.time()
    small = {1: (16, 32), 2: (24, 16), 3: (8, 16, 16), 4: (10, 12, 10)}
    for theta in ("gemm", "fft"):
        integrators.THETA_MODE = theta
        for k, dims in small.items():
            run_simulation(pcfg.BUILDERS[k](dims), 3, 3 * {1: 1e-3, 2: 1e-3, 3: 0.5, 4: 1e-2}[k])
        print(f"[{time.time() - t0:.0f}s] theta={theta}: configs 1-4", flush=True)
    integrators.THETA_MODE = "fft"
    cfgs = ["2", "7", "8", "9", "11", "12", "13"] if not quick else ["7", "8"]
    for cfg in cfgs:
        os.environ["CURVIGPU_TILE_CFG"] = cfg
        for k in (2, 4):
            run_simulation(pcfg.BUILDERS[k](small[k]), 2, 2e-3 if k == 2 else 2e-2)
    os.environ.pop("CURVIGPU_TILE_CFG", None)
    print(f"[{time.time() - t0:.0f}s] tile configs {cfgs}", flush=True)
    for chain in ("14", "15", None):
        if chain:
            os.environ.pop("CURVIGPU_NO_CHAIN", None)
            os.environ["CURVIGPU_CHAIN_CFG"] = chain
        else:
            os.environ["CURVIGPU_NO_CHAIN"] = "1"
        for dims in ((8, 16, 10), (5, 6, 7), (6, 8, 128)):
            run_simulation(pcfg.BUILDERS[4](dims), 2, 2e-2)
    os.environ.pop("CURVIGPU_NO_CHAIN", None)
    os.environ.pop("CURVIGPU_CHAIN_CFG", None)
    print(f"[{time.time() - t0:.0f}s] ball chain / two-stage", flush=True)
    # odd contiguous extents (padded storage, partial tiles)
    for k, dims in ((1, (5, 7)), (2, (7, 9)), (4, (5, 6, 7))):
        run_simulation(pcfg.BUILDERS[k](dims), 2, 2e-3 if k != 4 else 2e-2)
    # fused disk front in each CTA shape, lanes, on a small ensemble
    members = [pcfg.config5_member(i, (16, 32)) for i in range(0, 512, 37)]
    for variant in ({}, {"CURVIGPU_FRONT_NT256": "1"}, {"CURVIGPU_FRONT_NT64": "1"}):
        os.environ.update(variant)
        run_ensemble(members, 3, 3e-3)
        for key in variant:
            os.environ.pop(key)
    print(f"[{time.time() - t0:.0f}s] fused front variants", flush=True)
    # a 64-run ensemble at the real grid: 128-thread front CTAs, two lanes
    if not quick:
        big = [pcfg.config5_member(i, (128, 256)) for i in range(64)]
        run_ensemble(big, 2, 2e-3)
        print(f"[{time.time() - t0:.0f}s] 64-run 128x256 ensemble (lanes)", flush=True)
    # bulk-surface coupling + diagnostics reductions
    for name, dims in (("bulk_surface_schnakenberg_ball", {"n_rho": 6, "n_theta": 8, "n_phi": 6}),
                       ("bsdib_cylinder", {"n_rho": 6, "n_theta": 8, "n_z": 5})):
        sysm = models.build_system(name, dims, 1)
        run_simulation(sysm, 3, 3e-4, record_every=1, diagnostics=models.mean_diagnostics(sysm))
    sysm = pcfg.config1(small[1])
    run_simulation(sysm, 4, 4e-3, record_every=2, diagnostics=models.mean_diagnostics(sysm))
    torch.cuda.synchronize()
    print(f"[{time.time() - t0:.0f}s] sanitize workload done", flush=True)
    _ = np


if __name__ == "__main__":
    main()
