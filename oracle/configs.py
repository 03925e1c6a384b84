"""CPU ORACLE — test infrastructure only.  The five BASELINE.json configs
expressed through the oracle's restatement, at any
grid size so tests can shrink them.

Each builder returns an ``oracle.curvi_oracle.System``.  ``initial`` may be
supplied (e.g. the product's seeded fields, so both sides step identical
inputs); otherwise the oracle draws it with its own pure-Python xoshiro
(only sensible at small sizes).
"""

from __future__ import annotations

import numpy as np

from .curvi_oracle import (
    Comp,
    System,
    Xoshiro,
    anomalous_stencil,
    axial_stencil_nd,
    axial_stencil_nn,
    draw,
    fortran_fill,
    polar_stencil,
    radial_stencil,
    theta_stencil,
)

CONFIG_STEPS = {1: (1000, 1.0), 2: (2000, 2.0), 3: (500, 250.0), 4: (1000, 10.0), 5: (1000, 1.0)}
CONFIG_DIMS = {1: (64, 128), 2: (512, 256), 3: (64, 128, 128), 4: (100, 100, 100), 5: (128, 256)}


def _noise_ic(seed, shape, bases, law):
    rng = Xoshiro(seed)
    n = int(np.prod(shape))
    out = []
    for b in bases:
        f = np.full(shape, b)
        f += fortran_fill(draw(rng, law, n), shape)
        out.append(f)
    return out


def config1(dims=None, seed=1, initial=None):
    """Disk Schnakenberg."""
    n1, n2 = dims or CONFIG_DIMS[1]
    rho = radial_stencil(2, n1, 1.0)
    th = theta_stencil(n2)
    if initial is None:
        initial = _noise_ic(seed, (n1, n2), [1.0, 0.9], ("uniform", -1e-3, 1e-3))
    comps = [Comp("u", "disk", 1.0, rho=rho, theta=th, initial=initial[0]),
             Comp("v", "disk", 10.0, rho=rho, theta=th, initial=initial[1])]
    return System(comps, "schnakenberg", {"gamma": 100.0, "a": 0.1, "b": 0.9})


def config2(dims=None, seed=1, initial=None):
    """Sphere Brusselator; reference axis order (theta periodic, phi polar)."""
    n1, n2 = dims or CONFIG_DIMS[2]
    th = theta_stencil(n1)
    ph = polar_stencil(n2)
    A, B = 4.5, 6.96
    if initial is None:
        initial = _noise_ic(seed, (n1, n2), [A, B / A], ("uniform", -1e-2, 1e-2))
    comps = [Comp("u", "sphere", 0.01, theta=th, phi=ph, initial=initial[0]),
             Comp("v", "sphere", 0.08, theta=th, phi=ph, initial=initial[1])]
    return System(comps, "brusselator", {"A": A, "B": B})


def cylinder_box_ic(seed, shape, rho_grid, theta_grid, z_grid):
    """Config 3 initial state: u = 1, v = 0 plus a seeded box of half-width
    0.2 (centre r_c = 0.5 xi1, theta_c = 2 pi xi2, z_c = 0.3 + 1.4 xi3) set
    to u = 0.5(1 + 0.01 eta), v = 0.25(1 + 0.01 eta'), eta ~ U[-1, 1] drawn
    for every node in F order (u first, then v)."""
    rng = Xoshiro(seed)
    xi = rng.uniform(3)
    rc, tc, zc = 0.5 * xi[0], 2.0 * np.pi * xi[1], 0.3 + 1.4 * xi[2]
    n = int(np.prod(shape))
    eu = fortran_fill(draw(rng, ("uniform", -1.0, 1.0), n), shape)
    ev = fortran_fill(draw(rng, ("uniform", -1.0, 1.0), n), shape)
    R, T, Z = np.meshgrid(rho_grid, theta_grid, z_grid, indexing="ij")
    inside = ((np.abs(R * np.cos(T) - rc * np.cos(tc)) <= 0.2)
              & (np.abs(R * np.sin(T) - rc * np.sin(tc)) <= 0.2)
              & (np.abs(Z - zc) <= 0.2))
    u = np.where(inside, 0.5 * (1.0 + 0.01 * eu), 1.0)
    v = np.where(inside, 0.25 * (1.0 + 0.01 * ev), 0.0)
    return [u, v]


def config3(dims=None, seed=1, initial=None):
    """Cylinder Gray-Scott, Neumann walls and end caps, height 2."""
    n1, n2, n3 = dims or CONFIG_DIMS[3]
    rho = radial_stencil(2, n1, 1.0)
    th = theta_stencil(n2)
    z = axial_stencil_nn(n3, 2.0)
    if initial is None:
        initial = cylinder_box_ic(seed, (n1, n2, n3), rho.grid, th.grid, z.grid)
    comps = [Comp("u", "cylinder", 2e-5, rho=rho, theta=th, z=z, initial=initial[0]),
             Comp("v", "cylinder", 1e-5, rho=rho, theta=th, z=z, initial=initial[1])]
    return System(comps, "gray_scott", {"F": 0.04, "k": 0.06})


def config4(dims=None, seed=1, initial=None):
    """Ball BVAM (eta form); reference axis order (rho, theta periodic, phi polar)."""
    n1, n2, n3 = dims or CONFIG_DIMS[4]
    rho = radial_stencil(3, n1, 1.0)
    th = theta_stencil(n2)
    ph = polar_stencil(n3)
    if initial is None:
        initial = _noise_ic(seed, (n1, n2, n3), [0.0, 0.0], ("uniform", -1e-2, 1e-2))
    comps = [Comp("u", "ball", 0.516, rho=rho, theta=th, phi=ph, initial=initial[0]),
             Comp("v", "ball", 1.0, rho=rho, theta=th, phi=ph, initial=initial[1])]
    p = {"eta": 0.45, "a": 1.112, "b": -1.01, "h": -1.0, "C": 0.02}
    return System(comps, "bvam_eta", p)


def ensemble_gamma(i, runs=512):
    """gamma_i swept uniformly over [50, 200]."""
    return 50.0 + 150.0 * i / (runs - 1)


def config5_member(i, dims=None, runs=512, initial=None, lam=-1.95):
    """One ensemble member: the reference's schnakenberg_anomalous_disk
    (src/models.py:515-542) with alpha1 = gamma_i, alpha2 = 0.1,
    beta1 = 0.9, delta = 10, seed 1 + i; states are lifted."""
    n1, n2 = dims or CONFIG_DIMS[5]
    rho = anomalous_stencil(n1, 1.0, lam)
    weights = rho.grid ** (-2.0 - lam)
    th = theta_stencil(n2)
    ue = 0.1 + 0.9
    ve = 0.9 / ue**2
    if initial is None:
        f = _noise_ic(1 + i, (n1, n2), [ue, ve], ("normal", 1e-5))
        initial = [f[0] - ue, f[1] - ve]
    comps = [Comp("u", "disk", 1.0, rho=rho, theta=th, rho_weights=weights,
                  initial=initial[0], lift=ue),
             Comp("v", "disk", 10.0, rho=rho, theta=th, rho_weights=weights,
                  initial=initial[1], lift=ve)]
    return System(comps, "schnakenberg", {"gamma": ensemble_gamma(i, runs), "a": 0.1, "b": 0.9})


# published defaults of the two bulk-surface models (src/models.py:178-213)
BS_BALL_PARAMS = {"alpha1": 55.0, "alpha2": 0.1, "beta1": 0.9, "zeta1": 55.0, "zeta2": 5.0 / 12.0,
                  "zeta3": 5.0 / 12.0, "eta1": 5.0, "eta2": 5.0, "delta": 10.0, "epsilon": 10.0}
BS_CYL_PARAMS = {"alpha1": 1.0, "alpha2": 1.0, "alpha3": 0.15, "beta1": 1.0, "beta2": 1.0,
                 "beta3": 0.15, "delta": 1.0, "epsilon": 20.0, "zeta1": 1.0, "zeta2": 10.0,
                 "zeta3": 1.0, "zeta4": 66.0, "zeta5": 0.5, "eta1": 3.0, "eta2": 2.5,
                 "eta3": 0.2, "eta5": 1.5}


def bs_ball(dims, seed=1, initial=None, rho_star=1.0, params=None):
    """bulk_surface_schnakenberg_ball (src/models.py:570-611): ball u, v and
    sphere r, s, no lift; IC = equilibrium + Normal(1e-3) drawn u, v, r, s
    from one generator (src/models.py:236-237, :412-432).  ``dims`` =
    (n_rho, n_theta, n_phi)."""
    p = dict(BS_BALL_PARAMS, **(params or {}))
    n1, n2, n3 = dims
    rho = radial_stencil(3, n1, rho_star)
    th = theta_stencil(n2)
    ph = polar_stencil(n3)
    ue = p["alpha2"] + p["beta1"]
    ve = p["beta1"] / ue**2
    if initial is None:
        rng = Xoshiro(seed)
        initial = []
        for shape, base in (((n1, n2, n3), ue), ((n1, n2, n3), ve), ((n2, n3), ue), ((n2, n3), ve)):
            f = np.full(shape, base)
            f += fortran_fill(draw(rng, ("normal", 1e-3), int(np.prod(shape))), shape)
            initial.append(f)
    comps = [Comp("u", "ball", 1.0, rho=rho, theta=th, phi=ph, initial=initial[0]),
             Comp("v", "ball", p["delta"], rho=rho, theta=th, phi=ph, initial=initial[1]),
             Comp("r", "sphere", 1.0 / rho_star**2, theta=th, phi=ph, initial=initial[2]),
             Comp("s", "sphere", p["epsilon"] / rho_star**2, theta=th, phi=ph, initial=initial[3])]
    return System(comps, "bs_ball", dict(p, h=rho.h, rho_edge=rho.grid[-1]))


def bs_cylinder(dims, seed=1, initial=None, rho_star=25.0, z_star=25.0, params=None):
    """bsdib_cylinder (src/models.py:614-661): cylinder u, v (lifted by the
    equilibrium alpha2, beta2; no perturbation) and bottom-disk r, s
    (Uniform(0, 1e-2)).  ``dims`` = (n_rho, n_theta, n_z)."""
    p = dict(BS_CYL_PARAMS, **(params or {}))
    n1, n2, n3 = dims
    rho = radial_stencil(2, n1, rho_star)
    th = theta_stencil(n2)
    z = axial_stencil_nd(n3, z_star)
    ue, ve = p["alpha2"], p["beta2"]
    if initial is None:
        rng = Xoshiro(seed)
        initial = [np.zeros((n1, n2, n3)), np.zeros((n1, n2, n3))]
        for base in (0.0, p["zeta5"]):
            f = np.full((n1, n2), base)
            f += fortran_fill(draw(rng, ("uniform", 0.0, 1e-2), n1 * n2), (n1, n2))
            initial.append(f)
    comps = [Comp("u", "cylinder", 1.0, rho=rho, theta=th, z=z, initial=initial[0], lift=ue),
             Comp("v", "cylinder", p["delta"], rho=rho, theta=th, z=z, initial=initial[1], lift=ve),
             Comp("r", "disk", 1.0, rho=rho, theta=th, initial=initial[2]),
             Comp("s", "disk", p["epsilon"], rho=rho, theta=th, initial=initial[3])]
    return System(comps, "bs_cylinder", dict(p, h=z.h))


BUILDERS = {1: config1, 2: config2, 3: config3, 4: config4}
