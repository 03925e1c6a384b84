"""Systems for the engine: seeded initial fields, GPU kinetics descriptors,
and the reference's own disk/sphere models.

Mirrors the hot-path half of ``curvipat.models`` (models.py):
``Xoshiro256pp``/``Uniform``/``Normal`` (bit-exact, backed by C in
libcurvigpu.so), ``SystemComponent``, ``CoupledSystem``, ``model_spec``,
``build_system``, ``random_initial_condition``.  The reference's kinetics are
arbitrary Python closures (models.py:386-391); the engine instead takes a
:class:`Kinetics` descriptor naming one of the pointwise reactions compiled
into the F-build kernel.  The two bulk-surface models (models.py:322-369,
:570-661) carry a :class:`BulkSurfaceCoupling` descriptor instead, evaluated
by the coupling kernel (csrc/coupling.cuh) inside the coupled time loop
(paper_2604_11558_b200/coupled.py).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _native
from .integrators import ComponentOps, Geometry
from .operators import DiagonalWeights, build_lambda, build_phi_op, build_rho, build_theta, build_z

# ---------------------------------------------------------------------------
# seeded random numbers (models.py:43-130), C-backed
# ---------------------------------------------------------------------------


class Xoshiro256pp:
    """xoshiro256++ seeded by splitmix64; same stream as the reference."""

    def __init__(self, seed: int):
        self._state = (ctypes.c_uint64 * 4)()
        _native.lib().cg_rng_seed(ctypes.c_uint64(seed & (2**64 - 1)), self._state)

    def next_uint64(self) -> int:
        out = (ctypes.c_uint64 * 1)()
        _native.lib().cg_rng_next(self._state, 1, out)
        return int(out[0])

    def raw(self, size: int) -> np.ndarray:
        out = np.empty(size, dtype=np.uint64)
        _native.lib().cg_rng_next(self._state, size, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
        return out

    def uniform(self, size: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        out = np.empty(size)
        _native.lib().cg_rng_uniform(self._state, size, lo, hi, _native.dptr(out))
        return out

    def normal(self, size: int, sigma: float = 1.0) -> np.ndarray:
        out = np.empty(size)
        _native.lib().cg_rng_normal(self._state, size, sigma, _native.dptr(out))
        return out


@dataclass(frozen=True)
class Uniform:
    lo: float
    hi: float

    @property
    def scale(self) -> float:
        return (self.hi - self.lo) / math.sqrt(12.0)

    def draw(self, rng: Xoshiro256pp, size: int) -> np.ndarray:
        return rng.uniform(size, self.lo, self.hi)


@dataclass(frozen=True)
class Normal:
    sigma: float

    @property
    def scale(self) -> float:
        return self.sigma

    def draw(self, rng: Xoshiro256pp, size: int) -> np.ndarray:
        return rng.normal(size, self.sigma)


def unvec(w, dims):
    """First-index-fastest unflattening (tensor.py:24-28)."""
    return np.asarray(w).reshape(dims, order="F")


# ---------------------------------------------------------------------------
# kinetics descriptors
# ---------------------------------------------------------------------------

KINETICS_PARAMS = {
    "schnakenberg": ("gamma", "a", "b"),
    "brusselator": ("A", "B"),
    "gray_scott": ("F", "k"),
    "bvam_eta": ("eta", "a", "b", "h", "C"),
    "bvam": ("alpha1", "alpha2", "alpha3", "beta1", "beta2"),
    "dib": ("zeta1", "zeta2", "zeta3", "zeta4", "zeta5", "eta1", "eta2", "eta3", "eta5"),
}


@dataclass(frozen=True)
class Kinetics:
    """A pointwise two-species reaction the F-build kernel evaluates on the
    physical fields (lifted state + lift):

    - ``schnakenberg``: gamma(a - u + u^2 v), gamma(b - u^2 v)
      (models.py:293-296 scaled by alpha1 as in :528-532)
    - ``brusselator``: A - (B+1)u + u^2 v, B u - u^2 v
    - ``gray_scott``: -u v^2 + F(1-u), u v^2 - (F+k) v
    - ``bvam_eta``: eta(u + a v - C u v - u v^2), eta(b v + h u + C u v + u v^2)
    - ``bvam``: models.py:284-290
    - ``dib``: zeta1 * models.py:311-319 with eta4 from :299-308
    """

    kind: str
    params: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.kind not in KINETICS_PARAMS:
            raise NotImplementedError(f"no GPU kernel for kinetics {self.kind!r}")
        missing = [k for k in KINETICS_PARAMS[self.kind] if k not in self.params]
        if missing:
            raise ValueError(f"{self.kind} kinetics missing parameters {missing}")

    def param_vector(self) -> np.ndarray:
        return np.array([float(self.params[k]) for k in KINETICS_PARAMS[self.kind]])


BULK_SURFACE_PARAMS = {
    "ball": ("alpha1", "alpha2", "beta1", "zeta1", "zeta2", "zeta3", "eta1", "eta2"),
    "cylinder": ("alpha1", "alpha2", "alpha3", "beta1", "beta2", "beta3", "delta",
                 "zeta1", "zeta2", "zeta3", "zeta4", "zeta5", "eta1", "eta2", "eta3", "eta5"),
}


@dataclass(frozen=True)
class BulkSurfaceCoupling:
    """Reaction terms of a four-component bulk-surface system (bulk u, v;
    surface r, s), evaluated on the GPU from the common state:

    - ``ball``: alpha1 * Schnakenberg in the bulk plus the Robin ghost sources
      on the outermost rho slice, surface zeta1 * (Schnakenberg - exchange)
      (models.py:322-345, :587-602); ``h`` = h_rho, ``rho_edge`` = last rho node
    - ``cylinder``: linear bulk relaxation plus the flux sources on the z = 0
      slice, surface zeta1 * DIB with the v-dependent deposition term
      (models.py:348-369, :633-649); ``h`` = h_z
    """

    kind: str
    params: dict
    h: float
    rho_edge: float = 0.0

    def __post_init__(self):
        if self.kind not in BULK_SURFACE_PARAMS:
            raise NotImplementedError(f"no bulk-surface coupling {self.kind!r}")
        missing = [k for k in BULK_SURFACE_PARAMS[self.kind] if k not in self.params]
        if missing:
            raise ValueError(f"{self.kind} coupling missing parameters {missing}")

    def param_vector(self) -> np.ndarray:
        return np.array([float(self.params[k]) for k in BULK_SURFACE_PARAMS[self.kind]])


# ---------------------------------------------------------------------------
# the reference's own built-in kinetics closures -> descriptors
# ---------------------------------------------------------------------------

# qualname of the closure each reference builder returns (models.py:491-661)
_REFERENCE_CLOSURES = {
    "_build_bvam.<locals>.kinetics": "bvam_disk",
    "_build_anomalous.<locals>.kinetics": "schnakenberg_anomalous_disk",
    "_build_dib_sphere.<locals>.kinetics": "dib_sphere",
    "_build_ball.<locals>.kinetics": "bulk_surface_schnakenberg_ball",
    "_build_cylinder.<locals>.kinetics": "bsdib_cylinder",
}


def _closure_cells(fn) -> dict:
    names = getattr(getattr(fn, "__code__", None), "co_freevars", ())
    cells = getattr(fn, "__closure__", None) or ()
    out = {}
    for n, c in zip(names, cells):
        try:
            out[n] = c.cell_contents
        except ValueError:  # empty cell
            pass
    return out


def descriptor_for_model(name, params: dict, h: float | None = None, rho_edge: float | None = None):
    """The GPU descriptor of one of the reference's five built-in models
    (what each builder's closure computes, models.py:491-661): a
    :class:`Kinetics` for the two-species models, a
    :class:`BulkSurfaceCoupling` for the bulk-surface ones (``h`` = h_rho or
    h_z, ``rho_edge`` = last rho node of the ball)."""
    name = ModelName(name) if isinstance(name, str) else ModelName(getattr(name, "value", name))
    p = params
    if name is ModelName.BVAM_DISK:
        return Kinetics("bvam", {k: p[k] for k in KINETICS_PARAMS["bvam"]})
    if name is ModelName.SCHNAKENBERG_ANOMALOUS_DISK:
        return Kinetics("schnakenberg", {"gamma": p["alpha1"], "a": p["alpha2"], "b": p["beta1"]})
    if name is ModelName.DIB_SPHERE:
        return Kinetics("dib", {k: p[k] for k in KINETICS_PARAMS["dib"]})
    if name is ModelName.BULK_SURFACE_SCHNAKENBERG_BALL:
        return BulkSurfaceCoupling("ball", {k: p[k] for k in BULK_SURFACE_PARAMS["ball"]}, h=float(h),
                                   rho_edge=float(rho_edge))
    return BulkSurfaceCoupling("cylinder", {k: p[k] for k in BULK_SURFACE_PARAMS["cylinder"]}, h=float(h))


def reference_kinetics(system):
    """Descriptor for a system whose ``kinetics`` is one of the reference's
    own builder closures (``curvipat.models.build_system`` output), read
    from the closure itself -- its captured parameter map ``p`` and grid
    constants (h_rho, rho_edge, h_z) -- and cross-checked against
    ``system.spec``.  None for any other callable: an arbitrary Python
    closure has no GPU kernel."""
    fn = getattr(system, "kinetics", None)
    model = _REFERENCE_CLOSURES.get(getattr(fn, "__qualname__", ""))
    if model is None or not str(getattr(fn, "__module__", "")).endswith("models"):
        return None
    cells = _closure_cells(fn)
    p = cells.get("p")
    if not isinstance(p, dict):
        return None
    spec = getattr(system, "spec", None)
    spec_name = getattr(getattr(spec, "name", None), "value", None)
    if spec_name is not None and spec_name != model:
        return None
    try:
        if model == "bulk_surface_schnakenberg_ball":
            return descriptor_for_model(model, p, h=cells["h_rho"], rho_edge=cells["rho_edge"])
        if model == "bsdib_cylinder":
            return descriptor_for_model(model, p, h=cells["h_z"])
        return descriptor_for_model(model, p)
    except KeyError:
        return None


# ---------------------------------------------------------------------------
# systems
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class SystemComponent:
    """models.py:377-384."""

    name: str
    ops: object
    initial: np.ndarray
    lift: float = 0.0
    perturbation: object = None


@dataclass(frozen=True)
class CoupledSystem:
    """models.py:386-396, with ``kinetics`` a :class:`Kinetics` (or, for the
    bulk-surface models, :class:`BulkSurfaceCoupling`) descriptor."""

    spec: object
    components: list
    kinetics: Kinetics
    equilibrium: dict

    def physical_fields(self, states):
        lifts = {c.name: c.lift for c in self.components}
        return {name: W + lifts[name] for name, W in states.items()}


class ModelName(Enum):
    BVAM_DISK = "bvam_disk"
    SCHNAKENBERG_ANOMALOUS_DISK = "schnakenberg_anomalous_disk"
    DIB_SPHERE = "dib_sphere"
    BULK_SURFACE_SCHNAKENBERG_BALL = "bulk_surface_schnakenberg_ball"
    BSDIB_CYLINDER = "bsdib_cylinder"


# published defaults (models.py:148-221)
_DEFAULTS = {
    ModelName.BVAM_DISK: ({"gamma": 3.87e-3, "delta": 7.5e-3, "alpha1": 0.899, "alpha2": 0.2,
                           "alpha3": 0.2, "beta1": -0.91, "beta2": -0.899}, {"rho_star": 1.0}),
    ModelName.SCHNAKENBERG_ANOMALOUS_DISK: ({"alpha1": 5.0e2, "alpha2": 1.4e-1, "beta1": 1.34,
                                             "delta": 5.0e1, "lambda": -1.95}, {"rho_star": 1.0}),
    ModelName.DIB_SPHERE: ({"zeta1": 10.0, "zeta2": 10.0, "zeta3": 1.0, "zeta4": 48.0, "zeta5": 0.5,
                            "eta1": 5.0, "eta2": 2.5, "eta3": 0.2, "eta5": 1.5, "epsilon": 20.0},
                           {"rho_star": 1.1653}),
    ModelName.BULK_SURFACE_SCHNAKENBERG_BALL: ({"alpha1": 55.0, "alpha2": 0.1, "beta1": 0.9, "zeta1": 55.0,
                                                "zeta2": 5.0 / 12.0, "zeta3": 5.0 / 12.0, "eta1": 5.0,
                                                "eta2": 5.0, "delta": 10.0, "epsilon": 10.0},
                                               {"rho_star": 1.0}),
    ModelName.BSDIB_CYLINDER: ({"alpha1": 1.0, "alpha2": 1.0, "alpha3": 0.15, "beta1": 1.0, "beta2": 1.0,
                                "beta3": 0.15, "delta": 1.0, "epsilon": 20.0, "zeta1": 1.0, "zeta2": 10.0,
                                "zeta3": 1.0, "zeta4": 66.0, "zeta5": 0.5, "eta1": 3.0, "eta2": 2.5,
                                "eta3": 0.2, "eta5": 1.5}, {"rho_star": 25.0, "z_star": 25.0}),
}


@dataclass(frozen=True)
class ModelSpec:
    name: ModelName
    params: dict
    sizes: dict
    perturbations: dict

    def equilibrium(self) -> dict:
        p = self.params
        if self.name is ModelName.BVAM_DISK:
            return {"u": 0.0, "v": 0.0}
        if self.name is ModelName.SCHNAKENBERG_ANOMALOUS_DISK:
            ue = p["alpha2"] + p["beta1"]
            return {"u": ue, "v": p["beta1"] / ue**2}
        if self.name is ModelName.DIB_SPHERE:
            return {"r": 0.0, "s": p["zeta5"]}
        if self.name is ModelName.BULK_SURFACE_SCHNAKENBERG_BALL:
            ue = p["alpha2"] + p["beta1"]
            ve = p["beta1"] / ue**2
            return {"u": ue, "v": ve, "r": ue, "s": ve}
        return {"u": p["alpha2"], "v": p["beta2"], "r": 0.0, "s": p["zeta5"]}


def model_spec(name, overrides=None) -> ModelSpec:
    """models.py:247-276."""
    name = ModelName(name) if isinstance(name, str) else name
    params, sizes = (dict(x) for x in _DEFAULTS[name])
    for key, value in (overrides or {}).items():
        if key in sizes:
            sizes[key] = float(value)
        elif key in params:
            params[key] = float(value)
        else:
            raise KeyError(f"unknown parameter {key!r} for model {name.value}")
    if name is ModelName.BVAM_DISK:
        perts = {"u": Uniform(-0.5, 0.5), "v": Uniform(-0.5, 0.5)}
    elif name is ModelName.SCHNAKENBERG_ANOMALOUS_DISK:
        perts = {"u": Normal(1e-5), "v": Normal(1e-5)}
    elif name is ModelName.DIB_SPHERE:
        perts = {"r": Normal(1e-6), "s": Normal(1e-6)}
    elif name is ModelName.BULK_SURFACE_SCHNAKENBERG_BALL:
        perts = {c: Normal(1e-3) for c in ("u", "v", "r", "s")}
    else:
        perts = {"u": None, "v": None, "r": Uniform(0.0, 1e-2), "s": Uniform(0.0, 1e-2)}
    return ModelSpec(name, params, sizes, perts)


def component_shapes(name, dims: dict) -> dict:
    """Field dims per component (models.py:435-451)."""
    name = ModelName(name) if isinstance(name, str) else name
    if name in (ModelName.BVAM_DISK, ModelName.SCHNAKENBERG_ANOMALOUS_DISK):
        shape = (dims["n_rho"], dims["n_theta"])
        return {"u": shape, "v": shape}
    if name is ModelName.DIB_SPHERE:
        shape = (dims["n_theta"], dims["n_phi"])
        return {"r": shape, "s": shape}
    if name is ModelName.BULK_SURFACE_SCHNAKENBERG_BALL:
        bulk = (dims["n_rho"], dims["n_theta"], dims["n_phi"])
        surf = (dims["n_theta"], dims["n_phi"])
    else:
        bulk = (dims["n_rho"], dims["n_theta"], dims["n_z"])
        surf = (dims["n_rho"], dims["n_theta"])
    return {"u": bulk, "v": bulk, "r": surf, "s": surf}


def random_initial_condition(spec: ModelSpec, seed: int, dims: dict) -> dict:
    """Equilibrium + seeded perturbation, one generator, component-major, F
    order (models.py:412-432)."""
    rng = Xoshiro256pp(seed)
    shapes = component_shapes(spec.name, dims)
    eq = spec.equilibrium()
    out = {}
    for name, shape in shapes.items():
        base = np.full(shape, eq[name])
        law = spec.perturbations[name]
        if law is not None:
            base += unvec(law.draw(rng, int(np.prod(shape))), shape)
        out[name] = base
    return out


def _component(spec, name, ops, init, lift=0.0):
    return SystemComponent(name, ops, init[name] - lift, lift, spec.perturbations[name])


def build_system(spec, dims: dict, seed: int, overrides=None) -> CoupledSystem:
    """models.py:454-472 (builders :475-661), with GPU kinetics / coupling
    descriptors instead of closures."""
    if not isinstance(spec, ModelSpec):
        spec = model_spec(spec, overrides)
    elif overrides:
        raise ValueError("pass overrides via model_spec when supplying a ModelSpec")
    p = spec.params
    init = random_initial_condition(spec, seed, dims)
    eq = spec.equilibrium()
    if spec.name is ModelName.BVAM_DISK:
        rho = build_rho(2, dims["n_rho"], spec.sizes["rho_star"])
        theta = build_theta(dims["n_theta"])
        make = lambda k: ComponentOps(Geometry.DISK, k, rho=rho, theta=theta)  # noqa: E731
        comps = [_component(spec, "u", make(p["gamma"]), init), _component(spec, "v", make(p["delta"]), init)]
        kin = descriptor_for_model(spec.name, p)
    elif spec.name is ModelName.SCHNAKENBERG_ANOMALOUS_DISK:
        lam = p["lambda"]
        rho = build_lambda(dims["n_rho"], spec.sizes["rho_star"], lam)
        weights = DiagonalWeights(rho.grid ** (-2.0 - lam))
        theta = build_theta(dims["n_theta"])
        make = lambda k: ComponentOps(Geometry.DISK, k, rho=rho, theta=theta, rho_weights=weights)  # noqa: E731
        comps = [_component(spec, "u", make(1.0), init, eq["u"]),
                 _component(spec, "v", make(p["delta"]), init, eq["v"])]
        kin = descriptor_for_model(spec.name, p)
    elif spec.name is ModelName.DIB_SPHERE:
        rs = spec.sizes["rho_star"]
        theta = build_theta(dims["n_theta"])
        phi, _ = build_phi_op(dims["n_phi"])
        make = lambda k: ComponentOps(Geometry.SPHERE, k, theta=theta, phi=phi)  # noqa: E731
        comps = [_component(spec, "r", make(1.0 / rs**2), init),
                 _component(spec, "s", make(p["epsilon"] / rs**2), init)]
        kin = descriptor_for_model(spec.name, p)
    elif spec.name is ModelName.BULK_SURFACE_SCHNAKENBERG_BALL:
        # models.py:570-611
        rs = spec.sizes["rho_star"]
        rho = build_rho(3, dims["n_rho"], rs)
        theta = build_theta(dims["n_theta"])
        phi, _ = build_phi_op(dims["n_phi"])
        bulk = lambda k: ComponentOps(Geometry.BALL, k, rho=rho, theta=theta, phi=phi)  # noqa: E731
        surf = lambda k: ComponentOps(Geometry.SPHERE, k, theta=theta, phi=phi)  # noqa: E731
        comps = [_component(spec, "u", bulk(1.0), init), _component(spec, "v", bulk(p["delta"]), init),
                 _component(spec, "r", surf(1.0 / rs**2), init),
                 _component(spec, "s", surf(p["epsilon"] / rs**2), init)]
        kin = descriptor_for_model(spec.name, p, h=rho.h, rho_edge=rho.grid[-1])
    else:
        # models.py:614-661
        rho = build_rho(2, dims["n_rho"], spec.sizes["rho_star"])
        theta = build_theta(dims["n_theta"])
        z = build_z(dims["n_z"], spec.sizes["z_star"])
        bulk = lambda k: ComponentOps(Geometry.CYLINDER, k, rho=rho, theta=theta, z=z)  # noqa: E731
        surf = lambda k: ComponentOps(Geometry.DISK, k, rho=rho, theta=theta)  # noqa: E731
        comps = [_component(spec, "u", bulk(1.0), init, eq["u"]),
                 _component(spec, "v", bulk(p["delta"]), init, eq["v"]),
                 _component(spec, "r", surf(1.0), init), _component(spec, "s", surf(p["epsilon"]), init)]
        kin = descriptor_for_model(spec.name, p, h=z.h)
    return CoupledSystem(spec=spec, components=comps, kinetics=kin, equilibrium=eq)


# ---------------------------------------------------------------------------
# diagnostics (models.py:669-755); evaluated on the device by run_simulation /
# run_ensemble (cg_weighted_sums), on the host when called directly
# ---------------------------------------------------------------------------


def _clipped_widths(grid: np.ndarray, h: float, lo: float, hi: float) -> np.ndarray:
    """models.py:669-672."""
    left = np.clip(grid - h / 2.0, lo, hi)
    right = np.clip(grid + h / 2.0, lo, hi)
    return right - left


def _kind_name(op) -> str:
    k = getattr(op, "kind", None)
    return getattr(k, "value", k)


def quadrature_weights(cops, normalized: bool = True, rho_star: float | None = None) -> np.ndarray:
    """Node-centred quadrature weights with the coordinate Jacobian
    (models.py:675-715): truncated cells at the boundaries, normalised so the
    mean of a constant is exact.  Host setup, computed once per component."""
    g = getattr(cops.geometry, "value", cops.geometry)
    if g == "sphere":
        theta, phi = cops.theta, cops.phi
        radius = 1.0 if rho_star is None else rho_star
        wphi = _clipped_widths(phi.grid, phi.h, 0.0, np.pi)
        w = np.multiply.outer(np.full(theta.n, theta.h), radius**2 * np.sin(phi.grid) * wphi)
    else:
        rho = cops.rho
        edge = rho.grid[-1] + rho.h if _kind_name(rho) == "lambda" else rho.grid[-1]
        wrho = _clipped_widths(rho.grid, rho.h, 0.0, edge)
        theta_w = np.full(cops.theta.n, cops.theta.h)
        if g == "disk":
            w = np.multiply.outer(rho.grid * wrho, theta_w)
        elif g == "ball":
            phi = cops.phi
            wphi = _clipped_widths(phi.grid, phi.h, 0.0, np.pi)
            w = np.multiply.outer(np.multiply.outer(rho.grid**2 * wrho, theta_w), np.sin(phi.grid) * wphi)
        else:
            zop = cops.z
            wz = _clipped_widths(zop.grid, zop.h, 0.0, zop.grid[-1] + zop.h)
            w = np.multiply.outer(np.multiply.outer(rho.grid * wrho, theta_w), wz)
    return w / np.sum(w) if normalized else w


def integral_mean(field_values: np.ndarray, cops, rho_star: float | None = None) -> float:
    """Domain-averaged field value (models.py:718-725)."""
    w = quadrature_weights(cops, normalized=True, rho_star=rho_star)
    if np.shape(field_values) != w.shape:
        raise ValueError(f"field shape {np.shape(field_values)} does not match {w.shape}")
    return float(np.sum(field_values * w))


class MeanDiagnostics:
    """The closure of ``mean_diagnostics`` (models.py:728-744) as an object:
    called with a dict of host states it returns the physical integral mean
    of every component (the reference's behaviour); ``run_simulation`` and
    ``run_ensemble`` recognise it and evaluate it on the device instead, one
    weighted sum per component and sample (cg_weighted_sums), copying only
    the scalars back to the host."""

    def __init__(self, names, weights, lifts):
        self.names = list(names)
        self.weights = {n: np.ascontiguousarray(weights[n], dtype=np.float64) for n in self.names}
        self.lifts = {n: float(lifts[n]) for n in self.names}

    def __call__(self, states: dict) -> dict:
        return {name: float(np.sum(W * self.weights[name])) + self.lifts[name] for name, W in states.items()}

    def device_means(self, names, batch: int = 1) -> DeviceMeans:
        if list(names) != self.names:
            raise ValueError(f"diagnostics components {self.names} do not match the system's {list(names)}")
        return DeviceMeans([self.weights[n] for n in self.names], [self.lifts[n] for n in self.names], batch)


def mean_diagnostics(system) -> MeanDiagnostics:
    """models.py:728-744: quadrature weights built once, lifts restored."""
    spec = getattr(system, "spec", None)
    sizes = getattr(spec, "sizes", None) or {}
    rho_star = sizes.get("rho_star")
    names = [c.name for c in system.components]
    return MeanDiagnostics(
        names,
        {c.name: quadrature_weights(c.ops, normalized=True, rho_star=rho_star) for c in system.components},
        {c.name: getattr(c, "lift", 0.0) for c in system.components},
    )


class DeviceMeans:
    """Integral means of a device state [B][C][...]: out[b, c] =
    sum(W[b, c] * w[c]) + lift[c] by cg_weighted_sums (fixed summation order,
    graph-capturable, no host synchronisation)."""

    def __init__(self, weights, lifts, batch: int = 1):
        import torch

        self.C = len(weights)
        self.npts = int(np.asarray(weights[0]).size)
        if any(np.asarray(w).size != self.npts for w in weights):
            raise ValueError("every component needs weights of the same size")
        self.B = int(batch)
        self.w = torch.from_numpy(np.ascontiguousarray(np.stack([np.asarray(w, dtype=np.float64).ravel()
                                                                  for w in weights]))).to("cuda")
        self.off = torch.tensor([float(x) for x in lifts], dtype=torch.float64, device="cuda")
        L = _native.lib()
        n = L.cg_weighted_sums_scratch(self.B * self.C, self.npts)
        self.scratch = torch.empty(max(int(n), 1), dtype=torch.float64, device="cuda")

    def into(self, state, out) -> None:
        """Write the [B, C] means of ``state`` into the device tensor ``out``."""
        import torch

        if state.dtype != torch.float64 or not state.is_cuda or not state.is_contiguous():
            raise ValueError("state must be a contiguous float64 CUDA tensor")
        if state.numel() != self.B * self.C * self.npts:
            raise ValueError(f"state has {state.numel()} values, expected {self.B * self.C * self.npts}")
        if out.numel() != self.B * self.C or not out.is_contiguous() or out.dtype != torch.float64:
            raise ValueError("out must be a contiguous float64 tensor of B*C values")
        L = _native.lib()
        _native.check(L.cg_weighted_sums(state.data_ptr(), self.B * self.C, self.npts, self.w.data_ptr(), self.C,
                                         self.off.data_ptr(), out.data_ptr(), self.scratch.data_ptr(),
                                         self.scratch.numel(), torch.cuda.current_stream().cuda_stream),
                      "cg_weighted_sums")

    def __call__(self, state):
        import torch

        out = torch.empty((self.B, self.C), dtype=torch.float64, device="cuda")
        self.into(state, out)
        return out


def is_stabilized(times, values, rel: float = 1e-3, abs_tol: float = 1e-6) -> bool:
    """models.py:747-755."""
    times = np.asarray(times, dtype=float)
    values = np.asarray(values, dtype=float)
    t_star = times[-1]
    idx = int(np.argmin(np.abs(times - 0.9 * t_star)))
    return abs(values[-1] - values[idx]) <= rel * abs(values[-1]) + abs_tol
