"""Bulk-surface coupled time loop on the GPU.

The reference's two four-component models (models.py:570-661) couple a bulk
pair (u, v on a ball or cylinder) with a surface pair (r, s on the sphere or
the bottom disk) through the bulk trace.  run_simulation treats them like any
other system (integrators.py:413-427): per step the kinetics closure builds
every component's reaction term from the common state, then each component
takes one step_split.  Here that is one native call per chunk of steps
(``cg_coupled_run``): the coupling kernel evaluates all four reaction terms in
one pass, then the bulk plan and the surface plan (each a two-component
:class:`SplitPlan` with external G) step concurrently on two streams inside a
captured CUDA graph.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .integrators import INT32_MAX, DivergenceError, SplitPlan, prepare

_KIND = {"ball": _native.CG_BS_BALL, "cylinder": _native.CG_BS_CYLINDER}


class CoupledPlan:
    """Device state of one bulk-surface system: the bulk and surface plans,
    the coupling object and the four fields (lifted, as the reference
    integrates them).  Component order is (u, v, r, s) as in models.py."""

    def __init__(self, geos, coupling, lifts=None, theta: str | None = None):
        import torch

        geos = list(geos)
        if len(geos) != 4:
            raise ValueError("a bulk-surface system has four components (u, v, r, s)")
        lifts = [0.0] * 4 if lifts is None else [float(x) for x in lifts]
        self.coupling = coupling
        self.bulk = SplitPlan(geos[:2], batch=1, kinetics="external", lifts=lifts[:2], theta=theta)
        self.surf = SplitPlan(geos[2:], batch=1, kinetics="external", lifts=lifts[2:], theta=theta)
        if self.bulk.tau != self.surf.tau:
            raise ValueError("bulk and surface components must share tau")
        want = ("ball", "sphere") if coupling.kind == "ball" else ("cylinder", "disk")
        if (self.bulk.geometry, self.surf.geometry) != want:
            raise ValueError(f"{coupling.kind} coupling needs {want} components, got "
                             f"{(self.bulk.geometry, self.surf.geometry)}")
        self.tau = self.bulk.tau
        self._lib = _native.lib()
        params = np.ascontiguousarray(coupling.param_vector(), dtype=np.float64)
        d = _native.cg_coupling_desc()
        d.kind = _KIND[coupling.kind]
        for i, n in enumerate(self.bulk.shape):
            d.nb[i] = n
        sshape = self.surf.shape
        d.ns[0], d.ns[1] = sshape
        d.params = _native.dptr(params)
        d.nparams = params.size
        d.geom[0] = float(coupling.h)
        d.geom[1] = float(coupling.rho_edge)
        for i in range(4):
            d.lift[i] = lifts[i]
        handle = ctypes.c_void_p()
        _native.check(self._lib.cg_coupling_create(ctypes.byref(d), ctypes.byref(handle)), "cg_coupling_create")
        self._h = handle
        self.Wb = torch.zeros(self.bulk.state_shape, dtype=torch.float64, device="cuda")
        self.Ws = torch.zeros(self.surf.state_shape, dtype=torch.float64, device="cuda")
        self.first_bad = torch.full((4,), INT32_MAX, dtype=torch.int32, device="cuda")

    def close(self):
        if getattr(self, "_h", None):
            self._lib.cg_coupling_destroy(self._h)
            self._h = None
        for plan in (getattr(self, "bulk", None), getattr(self, "surf", None)):
            if plan is not None:
                plan.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _stream():
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def load(self, fields):
        """Upload the four (lifted) fields u, v, r, s."""
        import torch

        for dst, arrs in ((self.Wb, fields[:2]), (self.Ws, fields[2:])):
            host = np.ascontiguousarray(np.stack([np.asarray(a, dtype=np.float64) for a in arrs]))
            dst.copy_(torch.from_numpy(host).reshape(dst.shape))
        self.first_bad.fill_(INT32_MAX)

    def kinetics(self):
        """(Gb, Gs): the four reaction terms of the current state."""
        import torch

        Gb = torch.empty_like(self.Wb)
        Gs = torch.empty_like(self.Ws)
        _native.check(self._lib.cg_coupled_kinetics(self._h, self.Wb.data_ptr(), self.Ws.data_ptr(),
                                                    Gb.data_ptr(), Gs.data_ptr(), self._stream()),
                      "cg_coupled_kinetics")
        return Gb, Gs

    def run(self, step0: int, nsteps: int):
        """Advance the state by ``nsteps`` coupled steps numbered step0+1..."""
        _native.check(self._lib.cg_coupled_run(self._h, self.bulk._h, self.surf._h, self.Wb.data_ptr(),
                                               self.Ws.data_ptr(), int(step0), int(nsteps),
                                               self.first_bad.data_ptr(), self._stream()), "cg_coupled_run")

    def fields(self):
        """Device views of u, v, r, s (lifted)."""
        return [self.Wb[0, 0], self.Wb[0, 1], self.Ws[0, 0], self.Ws[0, 1]]

    def check_divergence(self, names):
        bad = self.first_bad.cpu().numpy()
        if bad.min() < INT32_MAX:
            s = int(bad.min())
            c = int(np.flatnonzero(bad == s)[0])
            raise DivergenceError(f"component {names[c]!r} diverged at step {s}", step=s)


def run_coupled(system, m: int, t_star: float, *, record_every=None, diagnostics=None, sample_hook=None,
                as_torch: bool = False, coupling=None):
    """run_simulation for a bulk-surface system (integrators.py:370-430);
    ``coupling`` is its BulkSurfaceCoupling (default: engine_kinetics)."""
    from .integrators import RunResult, engine_kinetics

    tau = t_star / m
    comps = list(system.components)
    names = [c.name for c in comps]
    coupling = coupling if coupling is not None else engine_kinetics(system)
    plan = CoupledPlan([prepare(c.ops, tau) for c in comps], coupling,
                       lifts=[float(getattr(c, "lift", 0.0)) for c in comps])
    plan.load([c.initial for c in comps])
    every = record_every or m
    times: list[float] = []
    series: dict[str, list[float]] = {n: [] for n in names}

    def host_states():
        return {n: f.cpu().numpy().copy() for n, f in zip(names, plan.fields())}

    def take_sample(step):
        t = step * tau
        times.append(t)
        if diagnostics is None and sample_hook is None:
            return
        st = host_states()
        if diagnostics is not None:
            for name, value in diagnostics(st).items():
                series[name].append(value)
        if sample_hook is not None:
            sample_hook(step, t, st)

    take_sample(0)
    step = 0
    while step < m:
        nxt = min(m, (step // every + 1) * every)
        plan.run(step, nxt - step)
        plan.check_divergence(names)
        step = nxt
        take_sample(step)
    if as_torch:
        fields = {n: f.clone() for n, f in zip(names, plan.fields())}
    else:
        fields = host_states()
    plan.close()
    return RunResult(fields=fields, times=times, series=series, steps=m, tau=tau)
