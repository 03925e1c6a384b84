"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
implementation (read-only at /root/reference/pkg/src) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (committed; small):
  rng.json         xoshiro256++ raw / Uniform / Normal streams
  setup.npz        operator bands, sigma, eigenpairs, phi1 values/tables
  steps.npz        apply_diffusion and step_split on random fields, all
                   geometries at small grids (incl. the reference tests' dims)
  runs.npz         run_simulation of the five BASELINE configs at reduced
                   grids (physical fields after m steps) + their ICs
  full.npz         the five BASELINE configs at FULL size: IC checksums and
                   strided samples / norms of the physical fields after
                   step 1 and step 100 (config 5: members 0, 255, 511)
  diagnostics.npz  quadrature_weights for every geometry / radial kind and
                   run_simulation(..., record_every, diagnostics=
                   mean_diagnostics(system)) series of the five BASELINE
                   configs at reduced grids
  converge.json    cmd_converge (cli.py:258-346) tables and slopes for three
                   built-in models at small grids (split-EE column)
  bulk_surface.npz the two bulk-surface models (models.py:570-661) through
                   model_spec/build_system/run_simulation: small grids in
                   full (IC, kinetics at the IC, state after 20 steps) and
                   the paper's full-size grids (samples after 1 and 100 steps)

The BASELINE systems are built through the reference's public API exactly as
SURVEY.md Appendix A prescribes (custom kinetics closures for configs 1-4,
the reference's own schnakenberg_anomalous_disk for config 5).
"""

from __future__ import annotations

import json
import math
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "8")
import numpy as np  # noqa: E402

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))

from curvipat import models, tensor  # noqa: E402
from curvipat import operators as op  # noqa: E402
from curvipat.integrators import (  # noqa: E402
    ComponentOps,
    Geometry,
    apply_diffusion,
    prepare,
    run_simulation,
    step_split,
)
from curvipat.models import CoupledSystem, SystemComponent, Uniform, Xoshiro256pp  # noqa: E402
from curvipat.phifun import phi1, phi1_matrix, phi1_outer  # noqa: E402

SAMPLES = 4096


# ---------------------------------------------------------------------------
# BASELINE configs through the reference API
# ---------------------------------------------------------------------------


from oracle.ref_configs import _noise, ref_config, ref_member, z_neumann  # noqa: E402,F401

STEPS = {1: (1000, 1.0), 2: (2000, 2.0), 3: (500, 250.0), 4: (1000, 10.0), 5: (1000, 1.0)}
FULL = {1: (64, 128), 2: (512, 256), 3: (64, 128, 128), 4: (100, 100, 100), 5: (128, 256)}
SMALL = {1: (16, 32), 2: (24, 16), 3: (8, 16, 16), 4: (10, 12, 10), 5: (16, 32)}


def physical(system, states):
    return {c.name: states[c.name] + c.lift for c in system.components}


# ---------------------------------------------------------------------------


def make_rng():
    out = {}
    for seed in (0, 1, 123, 2**63 + 5):
        r = Xoshiro256pp(seed)
        out[str(seed)] = {
            "raw": [str(r.next_uint64()) for _ in range(16)],
            "uniform": Uniform(-1e-3, 1e-3).draw(Xoshiro256pp(seed), 17).tolist(),
            "normal": models.Normal(1e-5).draw(Xoshiro256pp(seed), 17).tolist(),
        }
    (HERE / "rng.json").write_text(json.dumps(out, indent=1))


def make_setup():
    d = {}
    for n in (2, 3, 10, 64, 100, 256):
        d[f"sigma_{n}"] = np.array(op.solve_sigma(n))
        p, _ = op.build_phi_op(n)
        d[f"phi_{n}"] = np.stack([p.a, np.append(p.b, 0), np.append(p.c, 0), p.grid])
    for dd, n in ((2, 2), (2, 64), (3, 3), (3, 100), (2, 128)):
        r = op.build_rho(dd, n, 1.0)
        d[f"rho{dd}_{n}"] = np.stack([r.a, np.append(r.b, 0), np.append(r.c, 0), r.grid])
    for n, lam in ((128, -1.95), (16, -1.0), (8, 0.0)):
        r = op.build_lambda(n, 1.0, lam)
        d[f"lambda_{n}_{lam}"] = np.stack([r.a, np.append(r.b, 0), np.append(r.c, 0), r.grid])
    for n in (3, 4, 5, 8, 16):
        fac = op.eig_theta(op.build_theta(n))
        d[f"eigtheta_{n}_Q"] = fac.Q
        d[f"eigtheta_{n}_lam"] = fac.lambdas
    for name, o in (("rho2_64", op.build_rho(2, 64, 1.0)), ("phi_100", op.build_phi_op(100)[0]),
                    ("lambda_128", op.build_lambda(128, 1.0, -1.95)), ("z_16", op.build_z(16, 2.0))):
        fac = op.eig_tridiag(o)
        d[f"eig_{name}_lam"] = fac.lambdas
        d[f"eig_{name}_Vabs"] = np.abs(fac.V)  # column signs are LAPACK's choice
        d[f"eig_{name}_xi"] = fac.xi
        d[f"phi1m_{name}"] = phi1_matrix(0.0123, fac)
    x = np.concatenate([-np.logspace(-9, 2, 40), np.logspace(-9, 1.5, 40), [0.0, 1e-5, -1e-5, 9.99e-6]])
    d["phi1_x"] = x
    d["phi1_y"] = phi1(x)
    rs = np.random.RandomState(5)
    f1, f2, f3 = -rs.rand(5), -rs.rand(6) * 30, rs.rand(4)
    d["outer_f"] = np.concatenate([f1, f2, f3])
    d["outer2"] = phi1_outer(0.37, [f1, f2]).field
    d["outer3"] = phi1_outer(0.37, [f1, f2, f3]).field
    np.savez_compressed(HERE / "setup.npz", **d)


def _bases():
    return {
        "disk_4x4": ComponentOps(Geometry.DISK, 0.7, rho=op.build_rho(2, 4, 1.0), theta=op.build_theta(4)),
        "sphere_4x4": ComponentOps(Geometry.SPHERE, 0.9, theta=op.build_theta(4), phi=op.build_phi_op(4)[0]),
        "ball_3x4x4": ComponentOps(Geometry.BALL, 1.1, rho=op.build_rho(3, 3, 1.0), theta=op.build_theta(4),
                                   phi=op.build_phi_op(4)[0]),
        "cylinder_3x4x4": ComponentOps(Geometry.CYLINDER, 0.8, rho=op.build_rho(2, 3, 1.0),
                                       theta=op.build_theta(4), z=op.build_z(4, 1.0)),
        "disk_20x36": ComponentOps(Geometry.DISK, 1.3, rho=op.build_rho(2, 20, 1.0), theta=op.build_theta(36)),
        "adisk_33x64": ComponentOps(Geometry.DISK, 10.0, rho=op.build_lambda(33, 1.0, -1.95),
                                    theta=op.build_theta(64),
                                    rho_weights=op.DiagonalWeights(op.build_lambda(33, 1.0, -1.95).grid ** (-2.0 + 1.95))),
        "sphere_40x34": ComponentOps(Geometry.SPHERE, 0.08, theta=op.build_theta(40), phi=op.build_phi_op(34)[0]),
        "ball_12x10x18": ComponentOps(Geometry.BALL, 0.516, rho=op.build_rho(3, 12, 1.0),
                                      theta=op.build_theta(10), phi=op.build_phi_op(18)[0]),
        "cylinder_9x20x24": ComponentOps(Geometry.CYLINDER, 2e-2, rho=op.build_rho(2, 9, 1.0),
                                         theta=op.build_theta(20), z=z_neumann(24, 2.0)),
        "cylinderD_6x8x10": ComponentOps(Geometry.CYLINDER, 0.3, rho=op.build_rho(2, 6, 1.0),
                                         theta=op.build_theta(8), z=op.build_z(10, 1.5)),
        "ball_3x4x3": ComponentOps(Geometry.BALL, 1.1, rho=op.build_rho(3, 3, 1.0), theta=op.build_theta(4),
                                   phi=op.build_phi_op(3)[0]),
        "sphere_8x5": ComponentOps(Geometry.SPHERE, 0.9, theta=op.build_theta(8), phi=op.build_phi_op(5)[0]),
        "disk_5x7": ComponentOps(Geometry.DISK, 0.7, rho=op.build_rho(2, 5, 1.0), theta=op.build_theta(7)),
        "cylinder_3x4x5": ComponentOps(Geometry.CYLINDER, 0.8, rho=op.build_rho(2, 3, 1.0),
                                       theta=op.build_theta(4), z=op.build_z(5, 1.0)),
        "sphere_7x9": ComponentOps(Geometry.SPHERE, 0.3, theta=op.build_theta(7), phi=op.build_phi_op(9)[0]),
    }


def make_steps():
    d = {}
    rs = np.random.RandomState(22)
    for name, base in _bases().items():
        for tau in (0.037, 0.0):
            ops = prepare(base, tau)
            W = rs.randn(*base.shape)
            G = rs.randn(*base.shape)
            key = f"{name}_tau{tau}"
            d[key + "_W"] = W
            d[key + "_G"] = G
            d[key + "_MW"] = apply_diffusion(ops, W)
            d[key + "_out"] = step_split(ops, W, G)
    np.savez_compressed(HERE / "steps.npz", **d)


def make_runs():
    d = {}
    for k in (1, 2, 3, 4):
        sysm = ref_config(k, SMALL[k])
        m = 20
        t = STEPS[k][1] / STEPS[k][0] * m
        res = run_simulation(sysm, m, t)
        for c in sysm.components:
            d[f"c{k}_{c.name}_init"] = c.initial
            d[f"c{k}_{c.name}_final"] = physical(sysm, res.fields)[c.name]
        d[f"c{k}_m"] = np.array(m)
        d[f"c{k}_t"] = np.array(t)
    for i in (0, 7, 511):
        sysm = ref_member(i, SMALL[5])
        m = 20
        res = run_simulation(sysm, m, 0.02)
        for c in sysm.components:
            d[f"c5m{i}_{c.name}_init"] = c.initial
            d[f"c5m{i}_{c.name}_final"] = physical(sysm, res.fields)[c.name]
    np.savez_compressed(HERE / "runs.npz", **d)


def _sample_idx(n):
    return np.unique(np.linspace(0, n - 1, SAMPLES).astype(np.int64))


def _record(d, key, sysm, states):
    phys = physical(sysm, states)
    for c in sysm.components:
        f = phys[c.name].ravel()
        idx = _sample_idx(f.size)
        d[f"{key}_{c.name}_idx"] = idx
        d[f"{key}_{c.name}_val"] = f[idx]
        d[f"{key}_{c.name}_maxabs"] = np.array(np.max(np.abs(f)))
        d[f"{key}_{c.name}_sum"] = np.array(np.sum(f))


def make_full():
    d = {}
    for k in (1, 2, 3, 4):
        t0 = time.time()
        sysm = ref_config(k, FULL[k])
        m, ts = STEPS[k]
        tau = ts / m
        for c in sysm.components:
            d[f"f{k}_{c.name}_init_sum"] = np.array(np.sum(c.initial))
            d[f"f{k}_{c.name}_init_sample"] = c.initial.ravel()[_sample_idx(c.initial.size)]
        r1 = run_simulation(sysm, 1, tau)
        _record(d, f"f{k}_s1", sysm, r1.fields)
        r100 = run_simulation(sysm, 100, 100 * tau)
        _record(d, f"f{k}_s100", sysm, r100.fields)
        print(f"config {k}: {time.time() - t0:.1f}s", flush=True)
    for i in (0, 255, 511):
        sysm = ref_member(i, FULL[5])
        for c in sysm.components:
            d[f"f5m{i}_{c.name}_init_sum"] = np.array(np.sum(c.initial))
            d[f"f5m{i}_{c.name}_init_sample"] = c.initial.ravel()[_sample_idx(c.initial.size)]
        r1 = run_simulation(sysm, 1, 1e-3)
        _record(d, f"f5m{i}_s1", sysm, r1.fields)
        r100 = run_simulation(sysm, 100, 0.1)
        _record(d, f"f5m{i}_s100", sysm, r100.fields)
    np.savez_compressed(HERE / "full.npz", **d)


BS_CASES = {
    # name: (model, dims, m, t_star, seed, overrides)
    "ball_s": ("bulk_surface_schnakenberg_ball", {"n_rho": 6, "n_theta": 8, "n_phi": 6}, 20, 20 * 1e-4, 1, None),
    "ball_odd": ("bulk_surface_schnakenberg_ball", {"n_rho": 5, "n_theta": 10, "n_phi": 7}, 20, 20 * 1e-4, 3, None),
    "ball_zero": ("bulk_surface_schnakenberg_ball", {"n_rho": 4, "n_theta": 6, "n_phi": 4}, 20, 0.002, 9,
                  {"zeta2": 0.0, "zeta3": 0.0, "eta1": 0.0, "eta2": 0.0}),
    "cyl_s": ("bsdib_cylinder", {"n_rho": 6, "n_theta": 8, "n_z": 5}, 20, 20 * 6.25e-3, 1, None),
    "cyl_odd": ("bsdib_cylinder", {"n_rho": 7, "n_theta": 12, "n_z": 4}, 20, 20 * 6.25e-3, 4, None),
    # the paper's full-size runs (pkg/configs/ball_full.cfg, cylinder_full.cfg), 1 and 100 steps
    "ball_full": ("bulk_surface_schnakenberg_ball", {"n_rho": 30, "n_theta": 50, "n_phi": 30}, 100, 100 * 1e-4,
                  1, None),
    "cyl_full": ("bsdib_cylinder", {"n_rho": 160, "n_theta": 160, "n_z": 20}, 100, 100 * 6.25e-3, 1, None),
}


def make_bulk_surface():
    """bulk_surface.npz: the two bulk-surface models through the reference's
    own model_spec/build_system/run_simulation.  Small cases keep the whole
    fields (IC, kinetics at the IC, state after m steps); the full-size cases
    keep IC checksums and strided samples after 1 and m steps."""
    d = {}
    for key, (name, dims, m, t_star, seed, over) in BS_CASES.items():
        t0 = time.time()
        spec = models.model_spec(name, over)
        sysm = models.build_system(spec, dims, seed)
        full = key.endswith("_full")
        states0 = {c.name: c.initial for c in sysm.components}
        g0 = sysm.kinetics({k: v.copy() for k, v in states0.items()})
        for c in sysm.components:
            if full:
                d[f"{key}_{c.name}_init_sum"] = np.array(np.sum(c.initial))
                d[f"{key}_{c.name}_init_sample"] = c.initial.ravel()[_sample_idx(c.initial.size)]
            else:
                d[f"{key}_{c.name}_init"] = c.initial
                d[f"{key}_{c.name}_g0"] = g0[c.name]
        d[f"{key}_m"] = np.array(m)
        d[f"{key}_t"] = np.array(t_star)
        if full:
            r1 = run_simulation(sysm, 1, t_star / m)
            _record(d, f"{key}_s1", sysm, r1.fields)
            rm = run_simulation(sysm, m, t_star)
            _record(d, f"{key}_s{m}", sysm, rm.fields)
        else:
            res = run_simulation(sysm, m, t_star)
            for c in sysm.components:
                d[f"{key}_{c.name}_final"] = res.fields[c.name]
        print(f"{key}: {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(HERE / "bulk_surface.npz", **d)


DIAG_RUNS = {1: (23, 5), 2: (17, 4), 3: (9, 3), 4: (11, 4), 5: (20, 6)}  # (m, record_every)


def make_diagnostics():
    d = {}
    cases = {
        "disk": ComponentOps(Geometry.DISK, 1.0, rho=op.build_rho(2, 16, 1.0), theta=op.build_theta(32)),
        "disk_r2": ComponentOps(Geometry.DISK, 1.0, rho=op.build_rho(2, 9, 2.0), theta=op.build_theta(7)),
        "sphere": ComponentOps(Geometry.SPHERE, 1.0, theta=op.build_theta(12), phi=op.build_phi_op(9)[0]),
        "ball": ComponentOps(Geometry.BALL, 1.0, rho=op.build_rho(3, 10, 1.0), theta=op.build_theta(12),
                             phi=op.build_phi_op(10)[0]),
        "cylinder": ComponentOps(Geometry.CYLINDER, 1.0, rho=op.build_rho(2, 8, 1.0), theta=op.build_theta(16),
                                 z=op.build_z(16, 2.0)),
        "anomalous": ref_member(3, (16, 32)).components[0].ops,
    }
    for name, cops in cases.items():
        d[f"w_{name}"] = models.quadrature_weights(cops, normalized=True)
        d[f"wu_{name}"] = models.quadrature_weights(cops, normalized=False)
    d["wu_sphere_r"] = models.quadrature_weights(cases["sphere"], normalized=False, rho_star=1.1653)
    for k, (m, every) in DIAG_RUNS.items():
        sysm = ref_config(k, SMALL[k]) if k < 5 else ref_member(7, SMALL[5])
        t = STEPS[k][1] / STEPS[k][0] * m
        res = run_simulation(sysm, m, t, record_every=every, diagnostics=models.mean_diagnostics(sysm))
        d[f"c{k}_times"] = np.array(res.times)
        for c in sysm.components:
            d[f"c{k}_{c.name}_series"] = np.array(res.series[c.name])
    np.savez_compressed(HERE / "diagnostics.npz", **d)


CONVERGE_CASES = [
    {"model": "schnakenberg_anomalous_disk", "n_rho": 12, "n_theta": 16, "tstar": 0.002, "m_list": [5, 10, 20], "seed": 3},
    {"model": "bvam_disk", "n_rho": 10, "n_theta": 12, "tstar": 0.5, "m_list": [4, 8, 16], "m_ref": 96, "seed": 2},
    {"model": "dib_sphere", "n_theta": 12, "n_phi": 9, "tstar": 0.01, "m_list": [3, 6, 12], "seed": 5},
    {"model": "bulk_surface_schnakenberg_ball", "n_rho": 6, "n_theta": 8, "n_phi": 6, "tstar": 0.002,
     "m_list": [5, 10, 20], "seed": 4},
    {"model": "bsdib_cylinder", "n_rho": 6, "n_theta": 8, "n_z": 5, "tstar": 0.05, "m_list": [4, 8, 16], "seed": 6},
]


def make_converge():
    import contextlib
    import io

    from curvipat import cli

    out = []
    for cfg in CONVERGE_CASES:
        with contextlib.redirect_stdout(io.StringIO()):
            res = cli.cmd_converge(dict(cfg))
        out.append({"cfg": cfg, "table": res["table"], "slope": res["slope"]})
    (HERE / "converge.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    which = sys.argv[1:] or ["rng", "setup", "steps", "runs", "full", "bulk_surface", "diagnostics", "converge"]
    for w in which:
        t0 = time.time()
        globals()[f"make_{w}"]()
        print(f"{w}: {time.time() - t0:.1f}s", flush=True)
