"""Drop-in split exponential Euler engine on the B200.

Public surface mirrors the reference module ``curvipat.integrators``
(integrators.py): ``Geometry``, ``ComponentOps``, ``GeometryOps``,
``prepare``, ``apply_diffusion``, ``step_split``, ``STEPPERS``,
``run_simulation``, ``RunResult``, ``DivergenceError``,
``DIVERGENCE_LIMIT``.  ``prepare`` stays a host computation (north_star:
"operator assembly and the one-off phi1 evaluation ... may stay on the
host"); everything per step runs in libcurvigpu.so:

    apply_diffusion  -> cg_apply_diffusion (stencil kernel)
    step_split       -> cg_step            (F kernel + DMMA GEMM chain)
    run_simulation   -> cg_run             (CUDA-graph time loop, fused
                                             kinetics, on-device guard)

There is no CPU path: without a CUDA device or the built library these
functions raise.  Inputs are never mutated; numpy in -> numpy out, torch in
-> torch out (same device).  All work is ordered on the caller's current
torch CUDA stream.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from enum import Enum
from typing import Callable

import numpy as np

from . import _native
from .operators import (
    DiagonalWeights,
    EigenFactorization,
    PeriodicTridiagonal,
    TridiagonalOperator,
    eig_theta,
    eig_tridiag,
)
from .phifun import PhiTensor, phi1_matrix, phi1_outer

DIVERGENCE_LIMIT = 1e12  # integrators.py:33
INT32_MAX = 2**31 - 1


class DivergenceError(RuntimeError):
    """A field left the finite range; ``step`` is the 1-based step index
    (integrators.py:37-43)."""

    def __init__(self, message: str, step: int):
        super().__init__(message)
        self.step = step


class Geometry(Enum):
    DISK = "disk"
    SPHERE = "sphere"
    BALL = "ball"
    CYLINDER = "cylinder"


def _geometry_name(g) -> str:
    """Accept our Geometry, the reference's Geometry enum, or a string."""
    return g.value if isinstance(g, Enum) else str(g)


@dataclass(frozen=True)
class ComponentOps:
    """Geometry tag, diffusion coefficient and the 1-D operators of one
    component (integrators.py:53-84).  Reference ComponentOps objects are
    accepted everywhere this type is."""

    geometry: Geometry
    coeff: float
    rho: TridiagonalOperator | None = None
    theta: PeriodicTridiagonal | None = None
    phi: TridiagonalOperator | None = None
    z: TridiagonalOperator | None = None
    rho_weights: DiagonalWeights | None = None

    @property
    def shape(self) -> tuple[int, ...]:
        return _shape_of(self)

    def rho_weight_values(self):
        if self.rho is None:
            return None
        if self.rho_weights is not None:
            return self.rho_weights.values
        return self.rho.grid**-2.0


def _shape_of(base) -> tuple[int, ...]:
    g = _geometry_name(base.geometry)
    if g == "disk":
        return (base.rho.n, base.theta.n)
    if g == "sphere":
        return (base.theta.n, base.phi.n)
    if g == "ball":
        return (base.rho.n, base.theta.n, base.phi.n)
    return (base.rho.n, base.theta.n, base.z.n)


@dataclass(frozen=True)
class GeometryOps:
    """Per-(component, tau) operands built once by :func:`prepare`
    (integrators.py:87-127); host arrays, uploaded into a plan."""

    base: object
    tau: float
    A_rho: np.ndarray | None = None
    A_theta: np.ndarray | None = None
    A_phi: np.ndarray | None = None
    A_z: np.ndarray | None = None
    d_rho: np.ndarray | None = None
    d_phi: np.ndarray | None = None
    Q_theta: np.ndarray | None = None
    lam_theta: np.ndarray | None = None
    phi_fac: EigenFactorization | None = None
    phi_mix: PhiTensor | None = None
    phi_mix_outer: PhiTensor | None = None
    phi1_rho: np.ndarray | None = None
    phi1_phi: np.ndarray | None = None
    phi1_z: np.ndarray | None = None

    @property
    def geometry(self):
        return self.base.geometry

    @property
    def coeff(self) -> float:
        return self.base.coeff

    @property
    def shape(self) -> tuple[int, ...]:
        return _shape_of(self.base)


def _rho_weights(base):
    if base.rho is None:
        return None
    w = getattr(base, "rho_weights", None)
    if w is not None:
        return np.asarray(w.values, dtype=float)
    return base.rho.grid**-2.0


_OP_CACHE: dict = {}
_OP_CACHE_MAX = 64


def _op_key(op):
    parts = [type(op).__name__, getattr(op, "n", None), getattr(op, "h", None),
             str(getattr(op, "kind", ""))]
    for attr in ("a", "b", "c", "grid", "diag", "off"):
        v = getattr(op, attr, None)
        parts.append(None if v is None else np.asarray(v, dtype=np.float64).tobytes())
    return tuple(parts)


def _cached(op, what, fn):
    """Coefficient-independent setup of a 1-D operator (eigenpairs, dense
    copy), shared by every component / run that uses an operator with the
    same content -- a heterogeneous ensemble prepares one operator set per
    run, and these products are the same for all of them.  The results are
    read-only, as the reference treats prepared operands."""
    key = (what,) + _op_key(op)
    hit = _OP_CACHE.get(key)
    if hit is None:
        hit = fn(op)
        for arr in (hit if isinstance(hit, tuple) else (hit,)):
            for v in (vars(arr).values() if hasattr(arr, "__dict__") else (arr,)):
                if isinstance(v, np.ndarray):
                    v.flags.writeable = False
        if len(_OP_CACHE) >= _OP_CACHE_MAX:
            _OP_CACHE.pop(next(iter(_OP_CACHE)))
        _OP_CACHE[key] = hit
    return hit


def prepare(base, tau: float) -> GeometryOps:
    """Host setup of every transform and phi1 factor for one component at a
    fixed step (integrators.py:130-173).  Dense A_* copies are kept for API
    parity; the engine applies the stencils from the bands.  Eigenpairs and
    dense operator copies are cached by operator content (_cached): only the
    phi1 factors depend on tau * coeff."""
    if tau < 0:
        raise ValueError("tau must be nonnegative")
    g = _geometry_name(base.geometry)
    s = tau * base.coeff
    kw: dict = {}
    if base.theta is not None:
        fac = _cached(base.theta, "eig_theta", eig_theta)
        kw.update(A_theta=_cached(base.theta, "dense", lambda o: o.toarray()), Q_theta=fac.Q,
                  lam_theta=fac.lambdas)
    if base.rho is not None:
        kw.update(A_rho=_cached(base.rho, "dense", lambda o: o.toarray()), d_rho=_rho_weights(base),
                  phi1_rho=phi1_matrix(s, _cached(base.rho, "eig", eig_tridiag)))
    if base.phi is not None:
        fac = _cached(base.phi, "eig", eig_tridiag)
        kw.update(A_phi=_cached(base.phi, "dense", lambda o: o.toarray()),
                  d_phi=_cached(base.phi, "sin2", lambda o: np.sin(o.grid) ** -2.0), phi_fac=fac)
        if g == "sphere":
            kw["phi1_phi"] = phi1_matrix(s, fac)
    if base.z is not None:
        kw.update(A_z=_cached(base.z, "dense", lambda o: o.toarray()),
                  phi1_z=phi1_matrix(s, _cached(base.z, "eig", eig_tridiag)))
    if g == "disk":
        kw["phi_mix"] = phi1_outer(s, [kw["d_rho"], kw["lam_theta"]])
    elif g == "sphere":
        kw["phi_mix"] = phi1_outer(s, [kw["lam_theta"], kw["d_phi"]])
    elif g == "ball":
        kw["phi_mix_outer"] = phi1_outer(s, [kw["d_rho"], np.ones(base.theta.n), kw["phi_fac"].lambdas])
        kw["phi_mix"] = phi1_outer(s, [kw["d_rho"], kw["lam_theta"], kw["d_phi"]])
    elif g == "cylinder":
        kw["phi_mix"] = phi1_outer(s, [kw["d_rho"], kw["lam_theta"], np.ones(base.z.n)])
    else:
        raise ValueError(f"unknown geometry {g!r}")
    return GeometryOps(base=base, tau=tau, **kw)


# ---------------------------------------------------------------------------
# plan: host operands -> libcurvigpu
# ---------------------------------------------------------------------------

import os as _os

# How the periodic-theta factor Q diag(Phi) Q^T is applied: "gemm" = two dense
# DMMA mu-mode products (the reference's formulation), "fft" = the exact
# real-FFT propagator (csrc/thetafft.cuh).  Overridable per plan.
THETA_MODE = _os.environ.get("CURVIGPU_THETA", "fft")

KINETICS_CODES = {
    "external": 0,
    "schnakenberg": 1,
    "brusselator": 2,
    "gray_scott": 3,
    "bvam_eta": 4,
    "bvam": 5,
    "dib": 6,
}


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _bands(op) -> np.ndarray:
    out = np.zeros((3, op.n))
    out[0] = op.a
    out[1, :-1] = op.b
    out[2, :-1] = op.c
    return out


class SplitPlan:
    """A libcurvigpu plan for ``batch`` runs of a ``len(geos)``-component
    system whose components share geometry and grid.

    State tensors are torch.float64 CUDA tensors of shape
    ``(batch, ncomp, *grid)``, C-contiguous, reference axis order.
    """

    # runs per lane below which a plan is not split into lanes (auto mode).
    # Measured at the per-rank shard sizes of the 1/2/4/8-GPU ensemble
    # (profiles/r01_shard_sizes.jsonl): two lanes gain 1.5 % at 512 runs,
    # 6 % at 128 and 14 % at 64 runs (the 8-GPU shard), where one plan's
    # kernels run 1-2 ragged waves; 3 lanes add nothing (profiles/r01_lanes.txt)
    LANE_MIN_RUNS = 32

    def __init__(self, geos, batch: int = 1, kinetics: str = "external",
                 kin_params=None, lifts=None, theta: str | None = None, ops_per_run: bool = False,
                 lanes: int | None = None):
        """``geos``: one GeometryOps per component, shared by the ``batch``
        runs; with ``ops_per_run`` one per (run, component) in run-major
        order (a heterogeneous ensemble: runs may differ in coefficients and
        domain sizes, the grid extents must agree).

        ``lanes``: :meth:`run` advances the batch as that many independent
        sub-plans on their own streams (contiguous run blocks; runs never
        interact, so results are identical), which lets one lane's kernels
        fill the other's ragged kernel tails.  ``None`` picks 2 for batches of
        at least 2 * LANE_MIN_RUNS runs (env CURVIGPU_LANES overrides), else 1."""
        import torch  # noqa: F401  (device memory / streams)

        geos = list(geos)
        if not geos:
            raise ValueError("need at least one component")
        if ops_per_run and len(geos) % int(batch) != 0:
            raise ValueError("ops_per_run needs batch * ncomp operator sets")
        g = _geometry_name(geos[0].geometry)
        shape = tuple(geos[0].shape)
        taus = {float(o.tau) for o in geos}
        if any(_geometry_name(o.geometry) != g or tuple(o.shape) != shape for o in geos):
            raise NotImplementedError("components of one plan must share geometry and grid "
                                      "(bulk-surface systems run through coupled.CoupledPlan)")
        if len(taus) != 1:
            raise ValueError("components must share tau")
        if kinetics not in KINETICS_CODES:
            raise NotImplementedError(f"kinetics {kinetics!r} has no GPU kernel")
        self.geometry = g
        self.shape = shape
        self.batch = int(batch)
        self.ncomp = len(geos) // self.batch if ops_per_run else len(geos)
        self.ops_per_run = bool(ops_per_run)
        self.tau = taus.pop()
        C = self.ncomp
        keep = {}

        def stack(fn):
            arr = _f64(np.stack([fn(o) for o in geos]))
            keep[id(arr)] = arr
            return arr

        d = _native.cg_desc()
        d.geometry = _native.GEOMETRY_CODES[g]
        n = list(shape) + [1] * (3 - len(shape))
        d.n[0], d.n[1], d.n[2] = n
        d.batch = self.batch
        d.ncomp = C
        d.tau = self.tau
        coeff = stack(lambda o: o.coeff)
        d.coeff = _native.dptr(coeff)
        lift = _f64(np.zeros(C) if lifts is None else np.asarray(lifts, dtype=float))
        keep[id(lift)] = lift
        d.lift = _native.dptr(lift)
        base0 = geos[0].base
        if base0.theta is not None:
            d.theta_stencil = _native.dptr(stack(lambda o: [o.base.theta.diag, o.base.theta.off]))
            d.Q_theta = _native.dptr(stack(lambda o: o.Q_theta))
        if base0.rho is not None:
            d.rho_bands = _native.dptr(stack(lambda o: _bands(o.base.rho)))
            d.d_rho = _native.dptr(stack(lambda o: o.d_rho))
            d.phi1_rho = _native.dptr(stack(lambda o: o.phi1_rho))
        if base0.phi is not None:
            d.phi_bands = _native.dptr(stack(lambda o: _bands(o.base.phi)))
            d.d_phi = _native.dptr(stack(lambda o: o.d_phi))
        if base0.z is not None:
            d.z_bands = _native.dptr(stack(lambda o: _bands(o.base.z)))
            d.phi1_z = _native.dptr(stack(lambda o: o.phi1_z))
        if g == "sphere":
            d.phi1_phi = _native.dptr(stack(lambda o: o.phi1_phi))
        if g == "ball":
            d.V_phi = _native.dptr(stack(lambda o: o.phi_fac.V))
            d.Vinv_phi = _native.dptr(stack(lambda o: o.phi_fac.V_inv))
            d.Phi_outer = _native.dptr(stack(lambda o: o.phi_mix_outer.field[:, 0, :]))
            d.Phi = _native.dptr(stack(lambda o: o.phi_mix.field))
        elif g == "cylinder":
            d.Phi = _native.dptr(stack(lambda o: o.phi_mix.field[:, :, 0]))
        else:
            d.Phi = _native.dptr(stack(lambda o: o.phi_mix.field))
        d.kinetics = KINETICS_CODES[kinetics]
        self.kinetics = kinetics
        theta = theta or THETA_MODE
        if theta not in ("gemm", "fft"):
            raise ValueError(f"theta must be 'gemm' or 'fft', got {theta!r}")
        # 'fft' applies where n_theta is a power of two, else the plan keeps the GEMM pair
        self.theta = theta
        d.options = _native.CG_OPT_THETA_FFT if theta == "fft" else 0
        d.ops_per_run = 1 if ops_per_run else 0
        if kin_params is not None:
            kp = _f64(kin_params).reshape(self.batch, -1)
            keep[id(kp)] = kp
            d.nparams = kp.shape[1]
            d.kin_params = _native.dptr(kp)
        self._lib = _native.lib()
        handle = ctypes.c_void_p()
        _native.check(self._lib.cg_plan_create(ctypes.byref(d), ctypes.byref(handle)), "cg_plan_create")
        self._h = handle
        # lanes: sub-plans over contiguous run blocks (run() only)
        if lanes is None:
            env = os.environ.get("CURVIGPU_LANES")
            lanes = int(env) if env else (2 if self.batch >= 2 * self.LANE_MIN_RUNS else 1)
        lanes = max(1, min(int(lanes), self.batch))
        self._lanes = []
        if lanes > 1:
            kp_all = None if kin_params is None else _f64(kin_params).reshape(self.batch, -1)
            cuts = [self.batch * k // lanes for k in range(lanes + 1)]
            for lo, hi in zip(cuts[:-1], cuts[1:]):
                sub_geos = geos[lo * C:hi * C] if ops_per_run else geos
                sub = SplitPlan(sub_geos, batch=hi - lo, kinetics=kinetics,
                                kin_params=None if kp_all is None else kp_all[lo:hi], lifts=lifts,
                                theta=theta, ops_per_run=ops_per_run, lanes=1)
                self._lanes.append((lo, hi, sub, torch.cuda.Stream()))

    def close(self):
        for _, _, sub, _ in getattr(self, "_lanes", []):
            sub.close()
        self._lanes = []
        if getattr(self, "_h", None):
            self._lib.cg_plan_destroy(self._h)
            self._h = None

    @property
    def lanes(self) -> int:
        return max(1, len(self._lanes))

    def lane_blocks(self):
        """[(lo, hi, sub_plan, stream)] of the lanes (empty for one lane)."""
        return list(self._lanes)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers -------------------------------------------------------------
    @property
    def state_shape(self):
        return (self.batch, self.ncomp) + self.shape

    def _check_state(self, t, name):
        import torch

        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
            raise ValueError(f"{name} must be a CUDA float64 tensor")
        if tuple(t.shape) != self.state_shape or not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous with shape {self.state_shape}, got {tuple(t.shape)}")

    @staticmethod
    def _stream():
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    # -- entry points --------------------------------------------------------
    def apply_diffusion(self, W, out):
        self._check_state(W, "W")
        self._check_state(out, "out")
        _native.check(self._lib.cg_apply_diffusion(self._h, W.data_ptr(), out.data_ptr(), self._stream()),
                      "cg_apply_diffusion")

    def kinetics_into(self, W, G):
        self._check_state(W, "W")
        self._check_state(G, "G")
        _native.check(self._lib.cg_kinetics(self._h, W.data_ptr(), G.data_ptr(), self._stream()), "cg_kinetics")

    def step(self, W, G, out):
        self._check_state(W, "W")
        self._check_state(G, "G")
        self._check_state(out, "out")
        _native.check(self._lib.cg_step(self._h, W.data_ptr(), G.data_ptr(), out.data_ptr(), self._stream()),
                      "cg_step")

    # -- measurement access (bench.py) ---------------------------------------
    def stage_count(self) -> int:
        return int(self._lib.cg_plan_stage_count(self._h))

    def stage_info(self, stage: int) -> tuple[int, int]:
        """(algorithmic flops, algorithmic HBM bytes) of one launch of a
        stage; stage -1 is the F-build kernel."""
        fl, by = ctypes.c_longlong(), ctypes.c_longlong()
        _native.check(self._lib.cg_plan_stage_info(self._h, int(stage), ctypes.byref(fl), ctypes.byref(by)),
                      "cg_plan_stage_info")
        return int(fl.value), int(by.value)

    def step_kernels(self) -> list[int]:
        """Stage ids one cg_run step launches (-2 fused front, -1 F-build)."""
        ids = (ctypes.c_int * 32)()
        n = self._lib.cg_plan_step_kernels(self._h, ids, 32)
        if n < 0:
            _native.check(n, "cg_plan_step_kernels")
        return [ids[i] for i in range(min(n, 32))]

    def check_redzones(self) -> int:
        """Overwritten guard-band bytes around this plan's (and its lanes')
        workspaces; the plan must have been created with CURVIGPU_REDZONE=1."""
        total = 0
        for h in [self._h] + [sub._h for _, _, sub, _ in self._lanes]:
            n = int(self._lib.cg_plan_check_redzones(h))
            if n < 0:
                _native.check(n, "cg_plan_check_redzones")
            total += n
        return total

    def workspace(self, which: int):
        """Copy of workspace X (0), Y (1) or the second state buffer (2)."""
        import torch

        out = torch.empty(self.state_shape, dtype=torch.float64, device="cuda")
        _native.check(self._lib.cg_plan_copy_workspace(self._h, int(which), out.data_ptr(), self._stream()),
                      "cg_plan_copy_workspace")
        return out

    def run_stage(self, stage: int, W, out):
        self._check_state(W, "W")
        self._check_state(out, "out")
        _native.check(self._lib.cg_run_stage(self._h, int(stage), W.data_ptr(), out.data_ptr(), None,
                                             self._stream()), "cg_run_stage")

    def run(self, state, step0: int, nsteps: int, first_bad):
        """Advance ``state`` in place; ``first_bad`` is an int32 CUDA tensor
        of shape (batch, ncomp) receiving the first diverged step per field."""
        import torch

        self._check_state(state, "state")
        if first_bad.dtype != torch.int32 or not first_bad.is_cuda or first_bad.numel() != self.batch * self.ncomp:
            raise ValueError("first_bad must be an int32 CUDA tensor with batch*ncomp entries")
        if self._lanes:
            # fork: every lane waits for the caller's stream, runs its run block
            # on its own stream, and the caller's stream joins all lanes
            cur = torch.cuda.current_stream()
            ready = torch.cuda.Event()
            ready.record(cur)
            fb = first_bad.view(self.batch, self.ncomp)
            for lo, hi, sub, stream in self._lanes:
                stream.wait_event(ready)
                with torch.cuda.stream(stream):
                    sub.run(state[lo:hi], step0, nsteps, fb[lo:hi])
            for _, _, _, stream in self._lanes:
                cur.wait_stream(stream)
            return
        _native.check(self._lib.cg_run(self._h, state.data_ptr(), int(step0), int(nsteps), first_bad.data_ptr(),
                                       self._stream()), "cg_run")


# ---------------------------------------------------------------------------
# reference-shaped entry points
# ---------------------------------------------------------------------------

_PLAN_CACHE: dict[tuple, tuple[object, SplitPlan]] = {}


def _plan_for(ops) -> SplitPlan:
    key = (id(ops), THETA_MODE)
    hit = _PLAN_CACHE.get(key)
    if hit is not None and hit[0] is ops:
        return hit[1]
    plan = SplitPlan([ops], batch=1)
    if len(_PLAN_CACHE) > 64:
        _PLAN_CACHE.clear()
    _PLAN_CACHE[key] = (ops, plan)
    return plan


def _check_shape(x, shape):
    """The reference's shape check (integrators.py:178-179), done before any
    device work so a bad call fails the same way with or without a GPU."""
    got = tuple(x.shape) if hasattr(x, "shape") else np.shape(x)
    if tuple(got) != tuple(shape):
        raise ValueError(f"field shape {tuple(got)} does not match {tuple(shape)}")


def _to_device(x, shape):
    import torch

    if isinstance(x, torch.Tensor):
        if tuple(x.shape) != tuple(shape):
            raise ValueError(f"field shape {tuple(x.shape)} does not match {tuple(shape)}")
        return x.to(device="cuda", dtype=torch.float64).contiguous().reshape((1, 1) + tuple(shape)), True
    arr = np.asarray(x, dtype=np.float64)
    if arr.shape != tuple(shape):
        raise ValueError(f"field shape {arr.shape} does not match {tuple(shape)}")
    return torch.from_numpy(np.ascontiguousarray(arr)).to("cuda").reshape((1, 1) + tuple(shape)), False


def _from_device(t, shape, as_torch, like=None):
    out = t.reshape(tuple(shape))
    if as_torch:
        return out if like is None else out.to(like.device)
    return out.cpu().numpy()


def apply_diffusion(ops: GeometryOps, W):
    """coeff * M W on the GPU (integrators.py:176-199)."""
    import torch

    _check_shape(W, ops.shape)
    plan = _plan_for(ops)
    Wd, is_t = _to_device(W, ops.shape)
    out = torch.empty_like(Wd)
    plan.apply_diffusion(Wd, out)
    return _from_device(out, ops.shape, is_t, W if is_t else None)


def step_split(ops: GeometryOps, W, G):
    """One split exponential Euler step on the GPU (integrators.py:247-249)."""
    import torch

    _check_shape(W, ops.shape)
    _check_shape(G, ops.shape)
    plan = _plan_for(ops)
    Wd, is_t = _to_device(W, ops.shape)
    Gd, _ = _to_device(G, ops.shape)
    out = torch.empty_like(Wd)
    plan.step(Wd, Gd, out)
    return _from_device(out, ops.shape, is_t, W if is_t else None)


def _geometry_stepper(name):
    def stepper(ops, W, G):
        if _geometry_name(ops.geometry) != name:
            raise ValueError(f"{name} stepper got a {_geometry_name(ops.geometry)} operator")
        return step_split(ops, W, G)

    stepper.__name__ = f"step_split_{name}"
    return stepper


step_split_disk = _geometry_stepper("disk")
step_split_sphere = _geometry_stepper("sphere")
step_split_ball = _geometry_stepper("ball")
step_split_cylinder = _geometry_stepper("cylinder")

STEPPERS: dict[Geometry, Callable] = {
    Geometry.DISK: step_split_disk,
    Geometry.SPHERE: step_split_sphere,
    Geometry.BALL: step_split_ball,
    Geometry.CYLINDER: step_split_cylinder,
}


@dataclass
class RunResult:
    """Final (lifted) fields plus the sampled series (integrators.py:359-367)."""

    fields: dict
    times: list = field(default_factory=list)
    series: dict = field(default_factory=dict)
    steps: int = 0
    tau: float = 0.0


def engine_kinetics(system):
    """The GPU descriptor of a system's reaction terms: a ``models.Kinetics``
    (two-species systems) or ``models.BulkSurfaceCoupling`` (the
    bulk-surface models).  Accepted forms, in order: the descriptor itself as
    ``system.kinetics``; an ``engine_kinetics`` attribute; one of the
    reference's own builder closures (``curvipat.models.build_system``
    output: the descriptor is read from the closure, models.reference_kinetics).
    Any other Python callable raises NotImplementedError (it cannot run on the
    device, and there is no CPU fallback)."""
    from .models import BulkSurfaceCoupling, Kinetics, reference_kinetics

    for kin in (getattr(system, "kinetics", None), getattr(system, "engine_kinetics", None)):
        if isinstance(kin, (Kinetics, BulkSurfaceCoupling)):
            return kin
    kin = reference_kinetics(system)
    if kin is not None:
        return kin
    raise NotImplementedError(
        "system.kinetics is a Python callable the engine cannot run on the GPU: pass a "
        "paper_2604_11558_b200.models.Kinetics / BulkSurfaceCoupling descriptor (as system.kinetics or "
        "system.engine_kinetics), or a system built by curvipat.models.build_system (no CPU fallback)")


def _raise_if_diverged(bad, names):
    """DivergenceError for the first bad step, naming the first component (in
    component order) that diverged at it (integrators.py:422-427)."""
    if bad.min() < INT32_MAX:
        s = int(bad.min())
        c = int(np.flatnonzero(bad == s)[0])
        raise DivergenceError(f"component {names[c]!r} diverged at step {s}", step=s)


class _HostSampler:
    """Host copies of a [1][C][...] device state at sample steps for
    ``sample_hook`` and arbitrary diagnostics callables, overlapped with the
    next stepping chunk: ``stage`` snapshots the state on the device (and the
    divergence flags) and starts the download on a side stream; ``finish``
    waits for it, raises if the run had diverged by then, and returns the
    reference's dict of fresh arrays."""

    def __init__(self, state, first_bad, names):
        import torch

        self.state, self.first_bad, self.names = state, first_bad, names
        self.snap = torch.empty_like(state)
        self.host = torch.empty(state.shape, dtype=state.dtype, pin_memory=True)
        self.bad_dev = torch.empty_like(first_bad)
        self.bad = torch.empty(first_bad.shape, dtype=first_bad.dtype, pin_memory=True)
        self.side = torch.cuda.Stream()
        self.ready = torch.cuda.Event()
        self.done = torch.cuda.Event()

    def stage(self):
        import torch

        self.snap.copy_(self.state)
        self.bad_dev.copy_(self.first_bad)
        self.ready.record()
        with torch.cuda.stream(self.side):
            self.side.wait_event(self.ready)
            self.host.copy_(self.snap, non_blocking=True)
            self.bad.copy_(self.bad_dev, non_blocking=True)
            self.done.record(self.side)

    def finish(self) -> dict:
        self.done.synchronize()
        _raise_if_diverged(self.bad.numpy()[0], self.names)
        host = self.host.numpy()[0]
        return {n: host[i].copy() for i, n in enumerate(self.names)}


def run_simulation(system, m: int, t_star: float, *, record_every: int | None = None,
                   diagnostics: Callable | None = None, sample_hook: Callable | None = None,
                   method: str = "split", as_torch: bool = False) -> RunResult:
    """GPU run of a coupled system (integrators.py:370-430).

    Kinetics are evaluated from the common state before any component is
    updated; samples are taken at step 0, every ``record_every`` steps and at
    the final step; the divergence guard runs on the device after every step
    and raises ``DivergenceError(step)`` naming the first bad step and
    component, as the reference does.  ``diagnostics`` built by
    ``models.mean_diagnostics`` are evaluated on the device (only the scalars
    come back, once, at the end); a ``sample_hook`` or any other diagnostics
    callable gets host copies of the state, downloaded while the next chunk
    of steps runs.
    """
    import torch

    if m < 1:
        raise ValueError("need at least one time step")
    if t_star <= 0:
        raise ValueError("t_star must be positive")
    if method not in ("split", "forward_euler"):
        raise ValueError(f"unknown method {method!r}")
    if method != "split":
        raise NotImplementedError("forward Euler is a reference comparison path, not part of the engine")
    from .models import BulkSurfaceCoupling, Kinetics

    kin = engine_kinetics(system)
    if isinstance(kin, BulkSurfaceCoupling):
        from .coupled import run_coupled

        return run_coupled(system, m, t_star, record_every=record_every, diagnostics=diagnostics,
                           sample_hook=sample_hook, as_torch=as_torch, coupling=kin)
    if not isinstance(kin, Kinetics):
        raise NotImplementedError("two-species systems need a models.Kinetics descriptor")
    tau = t_star / m
    comps = list(system.components)
    names = [c.name for c in comps]
    geos = [prepare(c.ops, tau) for c in comps]
    lifts = [float(getattr(c, "lift", 0.0)) for c in comps]
    plan = SplitPlan(geos, batch=1, kinetics=kin.kind, kin_params=kin.param_vector()[None, :], lifts=lifts)
    state = torch.from_numpy(np.ascontiguousarray(np.stack([np.asarray(c.initial, dtype=np.float64)
                                                            for c in comps]))).to("cuda")
    state = state.reshape(plan.state_shape).contiguous()
    first_bad = torch.full((1, len(comps)), INT32_MAX, dtype=torch.int32, device="cuda")
    every = record_every or m
    # sample at step 0, every `every` steps and at m (integrators.py:413-430)
    sample_steps = [0]
    while sample_steps[-1] < m:
        sample_steps.append(min(m, (sample_steps[-1] // every + 1) * every))
    times = [k * tau for k in sample_steps]
    series: dict[str, list[float]] = {n: [] for n in names}
    from .models import MeanDiagnostics

    dev_diag = diagnostics if isinstance(diagnostics, MeanDiagnostics) else None
    host_diag = diagnostics if dev_diag is None else None
    sampler = _HostSampler(state, first_bad, names) if (host_diag is not None or sample_hook is not None) else None
    means = dev_diag.device_means(names, 1) if dev_diag is not None else None
    means_dev = (torch.empty((len(sample_steps), len(comps)), dtype=torch.float64, device="cuda")
                 if means is not None else None)

    def consume(i):
        st = sampler.finish()
        if host_diag is not None:
            for name, value in host_diag(st).items():
                series[name].append(value)
        if sample_hook is not None:
            sample_hook(sample_steps[i], times[i], st)

    # Stepping chunks are enqueued ahead: sample i's device means are written
    # by a kernel, its host copy (hooks / arbitrary diagnostics only) is
    # snapshotted on the device and downloaded on a side stream while chunk
    # i+1 runs; the divergence flags travel with it.
    if means is not None:
        means.into(state, means_dev[0])
    if sampler is not None:
        sampler.stage()
    for i in range(1, len(sample_steps)):
        plan.run(state, sample_steps[i - 1], sample_steps[i] - sample_steps[i - 1], first_bad)
        if means is not None:
            means.into(state, means_dev[i])
        if sampler is not None:
            consume(i - 1)
            sampler.stage()
    if sampler is not None:
        consume(len(sample_steps) - 1)
    _raise_if_diverged(first_bad.cpu().numpy()[0], names)
    if means is not None:
        vals = means_dev.cpu().numpy()
        for c, n in enumerate(names):
            series[n] = [float(x) for x in vals[:, c]]
    if as_torch:
        fields = {n: state[0, i].clone() for i, n in enumerate(names)}
    else:
        host = state[0].cpu().numpy()
        fields = {n: host[i].copy() for i, n in enumerate(names)}
    return RunResult(fields=fields, times=times, series=series, steps=m, tau=tau)
