"""CPU ORACLE infrastructure -- the BASELINE configs built through the REAL
reference's public API, for the golden-fixture
generator (tests/golden/make_golden.py, reference from /root/reference) and
for bench.py's reference arm / cpu_baseline (reference installed into the
git-ignored baseline/_ref, which travels to the GPU box).  Never product code.

Configs 1-4 have no reference builder: they are CoupledSystems with custom
kinetics closures over the reference's own operators and RNG (Appendix A);
config 5 members come from the reference's own build_system.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_DIR = ROOT / "baseline" / "_ref"


def load_curvipat(path=None):
    """Import curvipat from ``path`` (default: baseline/_ref, the installed
    reference); raises ImportError when it is absent."""
    path = Path(path) if path is not None else REF_DIR
    if not (path / "curvipat" / "__init__.py").exists():
        raise ImportError(f"curvipat not installed under {path}")
    if str(path) not in sys.path:
        sys.path.insert(0, str(path))
    import curvipat  # noqa: F401
    import curvipat.integrators  # noqa: F401
    import curvipat.models  # noqa: F401
    import curvipat.operators  # noqa: F401
    import curvipat.tensor  # noqa: F401

    return sys.modules["curvipat"]


def _api():
    from curvipat import models, tensor  # noqa: F401
    from curvipat import operators as op  # noqa: F401
    from curvipat.integrators import ComponentOps, Geometry  # noqa: F401
    from curvipat.models import CoupledSystem, SystemComponent, Uniform, Xoshiro256pp  # noqa: F401

    return models, tensor, op, ComponentOps, Geometry, CoupledSystem, SystemComponent, Uniform, Xoshiro256pp


def _noise(seed, shape, bases, law):
    models, tensor, op, ComponentOps, Geometry, CoupledSystem, SystemComponent, Uniform, Xoshiro256pp = _api()
    rng = Xoshiro256pp(seed)
    n = int(np.prod(shape))
    out = []
    for b in bases:
        f = np.full(shape, b)
        f += tensor.unvec(law.draw(rng, n), shape)
        out.append(f)
    return out


def z_neumann(n, height):
    op = _api()[2]
    h = height / (n - 1)
    b = np.full(n - 1, 1.0 / h**2)
    c = np.full(n - 1, 1.0 / h**2)
    b[0] = c[-1] = 2.0 / h**2
    return op.TridiagonalOperator(n=n, a=np.full(n, -2.0 / h**2), b=b, c=c, grid=h * np.arange(n), h=h,
                                  kind=op.OperatorKind.Z)


def ref_config(k, dims, seed=1):
    models, tensor, op, ComponentOps, Geometry, CoupledSystem, SystemComponent, Uniform, Xoshiro256pp = _api()
    spec = models.model_spec("bvam_disk")  # only read by diagnostics
    if k == 1:
        n1, n2 = dims
        rho, th = op.build_rho(2, n1, 1.0), op.build_theta(n2)
        u0, v0 = _noise(seed, (n1, n2), [1.0, 0.9], Uniform(-1e-3, 1e-3))
        g, a, b = 100.0, 0.1, 0.9

        def kin(s):
            u, v = s["u"], s["v"]
            uuv = u * u * v
            return {"u": g * (a - u + uuv), "v": g * (b - uuv)}

        comps = [SystemComponent("u", ComponentOps(Geometry.DISK, 1.0, rho=rho, theta=th), u0),
                 SystemComponent("v", ComponentOps(Geometry.DISK, 10.0, rho=rho, theta=th), v0)]
    elif k == 2:
        n1, n2 = dims
        th = op.build_theta(n1)
        ph, _ = op.build_phi_op(n2)
        A, B = 4.5, 6.96
        u0, v0 = _noise(seed, (n1, n2), [A, B / A], Uniform(-1e-2, 1e-2))

        def kin(s):
            u, v = s["u"], s["v"]
            uuv = u * u * v
            return {"u": A - (B + 1.0) * u + uuv, "v": B * u - uuv}

        comps = [SystemComponent("u", ComponentOps(Geometry.SPHERE, 0.01, theta=th, phi=ph), u0),
                 SystemComponent("v", ComponentOps(Geometry.SPHERE, 0.08, theta=th, phi=ph), v0)]
    elif k == 3:
        n1, n2, n3 = dims
        rho, th, z = op.build_rho(2, n1, 1.0), op.build_theta(n2), z_neumann(n3, 2.0)
        rng = Xoshiro256pp(seed)
        xi = rng.uniform(3)
        rc, tc, zc = 0.5 * xi[0], 2.0 * np.pi * xi[1], 0.3 + 1.4 * xi[2]
        n = n1 * n2 * n3
        eu = tensor.unvec(Uniform(-1.0, 1.0).draw(rng, n), dims)
        ev = tensor.unvec(Uniform(-1.0, 1.0).draw(rng, n), dims)
        R, T, Z = np.meshgrid(rho.grid, th.grid, z.grid, indexing="ij")
        inside = ((np.abs(R * np.cos(T) - rc * np.cos(tc)) <= 0.2)
                  & (np.abs(R * np.sin(T) - rc * np.sin(tc)) <= 0.2) & (np.abs(Z - zc) <= 0.2))
        u0 = np.where(inside, 0.5 * (1.0 + 0.01 * eu), 1.0)
        v0 = np.where(inside, 0.25 * (1.0 + 0.01 * ev), 0.0)
        F, kk = 0.04, 0.06

        def kin(s):
            u, v = s["u"], s["v"]
            uvv = u * v * v
            return {"u": -uvv + F * (1.0 - u), "v": uvv - (F + kk) * v}

        comps = [SystemComponent("u", ComponentOps(Geometry.CYLINDER, 2e-5, rho=rho, theta=th, z=z), u0),
                 SystemComponent("v", ComponentOps(Geometry.CYLINDER, 1e-5, rho=rho, theta=th, z=z), v0)]
    elif k == 4:
        n1, n2, n3 = dims
        rho, th = op.build_rho(3, n1, 1.0), op.build_theta(n2)
        ph, _ = op.build_phi_op(n3)
        u0, v0 = _noise(seed, dims, [0.0, 0.0], Uniform(-1e-2, 1e-2))
        eta, a, b, h, C = 0.45, 1.112, -1.01, -1.0, 0.02

        def kin(s):
            u, v = s["u"], s["v"]
            uv = u * v
            uvv = uv * v
            return {"u": eta * (u + a * v - C * uv - uvv), "v": eta * (b * v + h * u + C * uv + uvv)}

        comps = [SystemComponent("u", ComponentOps(Geometry.BALL, 0.516, rho=rho, theta=th, phi=ph), u0),
                 SystemComponent("v", ComponentOps(Geometry.BALL, 1.0, rho=rho, theta=th, phi=ph), v0)]
    else:
        raise ValueError(k)
    return CoupledSystem(spec=spec, components=comps, kinetics=kin, equilibrium={})


def ref_member(i, dims, runs=512):
    models = _api()[0]
    g = 50.0 + 150.0 * i / (runs - 1)
    spec = models.model_spec("schnakenberg_anomalous_disk",
                             {"alpha1": g, "alpha2": 0.1, "beta1": 0.9, "delta": 10.0})
    return models.build_system(spec, {"n_rho": dims[0], "n_theta": dims[1]}, 1 + i)


STEPS = {1: (1000, 1.0), 2: (2000, 2.0), 3: (500, 250.0), 4: (1000, 10.0), 5: (1000, 1.0)}
FULL = {1: (64, 128), 2: (512, 256), 3: (64, 128, 128), 4: (100, 100, 100), 5: (128, 256)}
