"""The five BASELINE.json workloads expressed through the engine's API
(SURVEY.md Appendix A).  Every builder takes optional smaller ``dims`` so
tests can shrink the grid without changing anything else.

Deviations from the BASELINE text, as documented in DESIGN.md:
- disk grids use the reference's half grid h = 1/(n - 1/2) (operators.py:172-201);
- BASELINE's (colatitude theta, longitude phi) is the reference's
  (phi, theta): the periodic axis comes first (integrators.py:69-77);
- config 3 uses a Neumann-Neumann axial stencil (operators.build_z_neumann)
  and a seeded box IC defined in :func:`cylinder_box_ic`;
- config 5 uses the reference's own schnakenberg_anomalous_disk build
  (lifted states, Normal(1e-5) IC) with seed_i = 1 + i and
  gamma_i = 50 + 150 i / (R - 1).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .integrators import ComponentOps, Geometry
from .models import CoupledSystem, Kinetics, SystemComponent, Xoshiro256pp, build_system, model_spec, unvec
from .operators import build_phi_op, build_rho, build_theta, build_z_neumann

STEPS = {1: (1000, 1.0), 2: (2000, 2.0), 3: (500, 250.0), 4: (1000, 10.0), 5: (1000, 1.0)}
DIMS = {1: (64, 128), 2: (512, 256), 3: (64, 128, 128), 4: (100, 100, 100), 5: (128, 256)}
ENSEMBLE_RUNS = 512
NAMES = {1: "disk_schnakenberg_64x128", 2: "sphere_brusselator_512x256", 3: "cylinder_grayscott_64x128x128",
         4: "ball_bvam_100x100x100", 5: "ensemble512_anomalous_disk_128x256"}


def _noise(seed, shape, bases, law):
    rng = Xoshiro256pp(seed)
    n = int(np.prod(shape))
    fields = []
    for b in bases:
        f = np.full(shape, b)
        f += unvec(law.draw(rng, n), shape)
        fields.append(f)
    return fields


def _system(comps, kin, spec=None):
    return CoupledSystem(spec=spec, components=comps, kinetics=kin, equilibrium={})


def config1(dims=None, seed=1) -> CoupledSystem:
    """Disk, Schnakenberg a=0.1, b=0.9, d=10, gamma=100; U[-1e-3, 1e-3] noise."""
    from .models import Uniform

    n1, n2 = dims or DIMS[1]
    rho, th = build_rho(2, n1, 1.0), build_theta(n2)
    u0, v0 = _noise(seed, (n1, n2), [1.0, 0.9], Uniform(-1e-3, 1e-3))
    comps = [SystemComponent("u", ComponentOps(Geometry.DISK, 1.0, rho=rho, theta=th), u0),
             SystemComponent("v", ComponentOps(Geometry.DISK, 10.0, rho=rho, theta=th), v0)]
    return _system(comps, Kinetics("schnakenberg", {"gamma": 100.0, "a": 0.1, "b": 0.9}))


def config2(dims=None, seed=1) -> CoupledSystem:
    """Sphere, Brusselator A=4.5, B=6.96, D_u=0.01, D_v=0.08; (512 periodic, 256 polar)."""
    from .models import Uniform

    n1, n2 = dims or DIMS[2]
    th = build_theta(n1)
    ph, _ = build_phi_op(n2)
    A, B = 4.5, 6.96
    u0, v0 = _noise(seed, (n1, n2), [A, B / A], Uniform(-1e-2, 1e-2))
    comps = [SystemComponent("u", ComponentOps(Geometry.SPHERE, 0.01, theta=th, phi=ph), u0),
             SystemComponent("v", ComponentOps(Geometry.SPHERE, 0.08, theta=th, phi=ph), v0)]
    return _system(comps, Kinetics("brusselator", {"A": A, "B": B}))


def cylinder_box_ic(seed, shape, rho_grid, theta_grid, z_grid):
    """u = 1, v = 0 plus a seeded box of half-width 0.2: centre
    (r_c, theta_c, z_c) = (0.5 xi1, 2 pi xi2, 0.3 + 1.4 xi3); inside it
    u = 0.5(1 + 0.01 eta), v = 0.25(1 + 0.01 eta'), eta ~ U[-1, 1] drawn for
    every node in F order, u first."""
    from .models import Uniform

    rng = Xoshiro256pp(seed)
    xi = rng.uniform(3)
    rc, tc, zc = 0.5 * xi[0], 2.0 * np.pi * xi[1], 0.3 + 1.4 * xi[2]
    n = int(np.prod(shape))
    law = Uniform(-1.0, 1.0)
    eu = unvec(law.draw(rng, n), shape)
    ev = unvec(law.draw(rng, n), shape)
    R, T, Z = np.meshgrid(rho_grid, theta_grid, z_grid, indexing="ij")
    inside = ((np.abs(R * np.cos(T) - rc * np.cos(tc)) <= 0.2)
              & (np.abs(R * np.sin(T) - rc * np.sin(tc)) <= 0.2)
              & (np.abs(Z - zc) <= 0.2))
    return np.where(inside, 0.5 * (1.0 + 0.01 * eu), 1.0), np.where(inside, 0.25 * (1.0 + 0.01 * ev), 0.0)


def config3(dims=None, seed=1) -> CoupledSystem:
    """Cylinder (radius 1, height 2), Gray-Scott D_u=2e-5, D_v=1e-5, F=0.04, k=0.06."""
    n1, n2, n3 = dims or DIMS[3]
    rho, th, z = build_rho(2, n1, 1.0), build_theta(n2), build_z_neumann(n3, 2.0)
    u0, v0 = cylinder_box_ic(seed, (n1, n2, n3), rho.grid, th.grid, z.grid)
    comps = [SystemComponent("u", ComponentOps(Geometry.CYLINDER, 2e-5, rho=rho, theta=th, z=z), u0),
             SystemComponent("v", ComponentOps(Geometry.CYLINDER, 1e-5, rho=rho, theta=th, z=z), v0)]
    return _system(comps, Kinetics("gray_scott", {"F": 0.04, "k": 0.06}))


def config4(dims=None, seed=1) -> CoupledSystem:
    """Ball (rho, theta periodic, phi polar), BVAM eta-form, D=0.516."""
    from .models import Uniform

    n1, n2, n3 = dims or DIMS[4]
    rho, th = build_rho(3, n1, 1.0), build_theta(n2)
    ph, _ = build_phi_op(n3)
    u0, v0 = _noise(seed, (n1, n2, n3), [0.0, 0.0], Uniform(-1e-2, 1e-2))
    comps = [SystemComponent("u", ComponentOps(Geometry.BALL, 0.516, rho=rho, theta=th, phi=ph), u0),
             SystemComponent("v", ComponentOps(Geometry.BALL, 1.0, rho=rho, theta=th, phi=ph), v0)]
    return _system(comps, Kinetics("bvam_eta", {"eta": 0.45, "a": 1.112, "b": -1.01, "h": -1.0, "C": 0.02}))


def ensemble_gamma(i: int, runs: int = ENSEMBLE_RUNS) -> float:
    return 50.0 + 150.0 * i / (runs - 1)


def config5_member(i: int, dims=None, runs: int = ENSEMBLE_RUNS) -> CoupledSystem:
    """Member i of the ensemble: the reference's schnakenberg_anomalous_disk
    with alpha1 = gamma_i, alpha2 = 0.1, beta1 = 0.9, delta = 10, seed 1+i."""
    n1, n2 = dims or DIMS[5]
    spec = model_spec("schnakenberg_anomalous_disk",
                      {"alpha1": ensemble_gamma(i, runs), "alpha2": 0.1, "beta1": 0.9, "delta": 10.0})
    return build_system(spec, {"n_rho": n1, "n_theta": n2}, 1 + i)


@dataclass
class EnsembleInputs:
    """Batched ensemble inputs: states [R, 2, n1, n2] (lifted) and gammas [R]."""

    template: CoupledSystem  # member 0 (operators shared by all members)
    states: np.ndarray
    gammas: np.ndarray
    first: int


def config5_inputs(first: int, count: int, dims=None, runs: int = ENSEMBLE_RUNS) -> EnsembleInputs:
    """Members first .. first+count-1, built on the host (ICs from the C RNG)."""
    members = [config5_member(i, dims, runs) for i in range(first, first + count)]
    states = np.stack([np.stack([c.initial for c in s.components]) for s in members])
    gammas = np.array([ensemble_gamma(i, runs) for i in range(first, first + count)])
    return EnsembleInputs(members[0], states, gammas, first)


BUILDERS = {1: config1, 2: config2, 3: config3, 4: config4}
