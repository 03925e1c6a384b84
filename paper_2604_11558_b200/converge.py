"""Time-step convergence study on the GPU: the split-EE column of the
reference's ``curvipat converge`` (cmd_converge, cli.py:258-346).

The reference runs ``run_simulation`` once at m_ref and once per m in
m_list, one after another, and fits the slope of log(err) against log(m).
Here every run gets its own plan (tau differs, so operators differ) and its
own CUDA stream, so the runs execute concurrently; the errors use the
reference's formula (_relative_error, cli.py:250-255) on the lifted fields
that run_simulation returns.  The CLI, printing, CSV output and the dense /
forward-Euler comparison columns are out of scope.
"""

from __future__ import annotations

import math

import numpy as np

from .integrators import INT32_MAX, DivergenceError, SplitPlan, engine_kinetics, prepare
from .coupled import CoupledPlan
from .models import BulkSurfaceCoupling, build_system


def relative_error(states: dict, reference: dict) -> float:
    """cli.py:250-255: sqrt(sum_c (|W_c - ref_c| / |ref_c|)^2), Frobenius norms."""
    total = 0.0
    for name, ref in reference.items():
        diff = np.linalg.norm(states[name] - ref)
        total += (diff / np.linalg.norm(ref)) ** 2
    return math.sqrt(total)


def convergence_study(spec, dims: dict, t_star: float, m_list, *, m_ref: int | None = None,
                      seed: int = 1) -> dict:
    """Split-EE errors against an m_ref-step reference solution for every m in
    ``m_list`` (ascending) and the least-squares slope of log(err) vs log(m).
    Returns ``{"table": [{"m": m, "err_split": e}, ...], "slope": s}`` like
    cmd_converge.  Raises ValueError for a bad m_list / m_ref (the CLI's
    UsageError) and DivergenceError if any run diverges."""
    import torch

    m_list = [int(m) for m in m_list]
    if not m_list:
        raise ValueError("m_list must not be empty")
    if sorted(m_list) != m_list:
        raise ValueError("m_list must be ascending")
    if m_ref is None:
        m_ref = 4 * max(m_list)
    if m_ref < 4 * max(m_list):
        raise ValueError("reference step count must be at least 4x max(m_list)")
    if t_star <= 0 or min(m_list) < 1:
        raise ValueError("t_star must be positive and every m >= 1")

    system = build_system(spec, dims, seed)
    kin = engine_kinetics(system)
    if isinstance(kin, BulkSurfaceCoupling):
        fields = _coupled_runs(system, kin, t_star, [m_ref] + m_list)
        return _table(m_list, fields)
    comps = list(system.components)
    names = [c.name for c in comps]
    lifts = [float(getattr(c, "lift", 0.0)) for c in comps]
    init = np.ascontiguousarray(np.stack([np.asarray(c.initial, dtype=np.float64) for c in comps]))
    runs = []
    for m in [m_ref] + m_list:
        tau = t_star / m
        plan = SplitPlan([prepare(c.ops, tau) for c in comps], batch=1, kinetics=kin.kind,
                         kin_params=kin.param_vector()[None, :], lifts=lifts)
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            state = torch.from_numpy(init).to("cuda", non_blocking=False).reshape(plan.state_shape).contiguous()
            bad = torch.full((1, len(comps)), INT32_MAX, dtype=torch.int32, device="cuda")
            plan.run(state, 0, m, bad)
        runs.append((m, plan, stream, state, bad))
    fields = []
    for m, plan, stream, state, bad in runs:
        stream.synchronize()
        b = bad.cpu().numpy()[0]
        if b.min() < INT32_MAX:
            s = int(b.min())
            c = int(np.flatnonzero(b == s)[0])
            raise DivergenceError(f"component {names[c]!r} diverged at step {s} (m = {m})", step=s)
        host = state[0].cpu().numpy()
        fields.append({n: host[i].copy() for i, n in enumerate(names)})
        plan.close()
    return _table(m_list, fields)


def _table(m_list, fields) -> dict:
    """cmd_converge's table and slope from the m_ref run (fields[0]) and the
    m_list runs (cli.py:286-312)."""
    reference = fields[0]
    table = [{"m": m, "err_split": relative_error(f, reference)} for m, f in zip(m_list, fields[1:])]
    slope = float(np.polyfit(np.log([e["m"] for e in table]), np.log([e["err_split"] for e in table]), 1)[0])
    return {"table": table, "slope": slope}


def _coupled_runs(system, coupling, t_star: float, ms) -> list:
    """The bulk-surface models (ball + sphere, cylinder + disk): one
    CoupledPlan per m, each on its own stream so the runs overlap; lifted
    fields per run, DivergenceError as run_simulation raises it."""
    import torch

    comps = list(system.components)
    names = [c.name for c in comps]
    lifts = [float(getattr(c, "lift", 0.0)) for c in comps]
    runs = []
    for m in ms:
        tau = t_star / m
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            plan = CoupledPlan([prepare(c.ops, tau) for c in comps], coupling, lifts=lifts)
            plan.load([c.initial for c in comps])
            plan.run(0, m)
        runs.append((m, plan, stream))
    fields = []
    for m, plan, stream in runs:
        stream.synchronize()
        plan.check_divergence(names)
        fields.append({n: f.cpu().numpy().copy() for n, f in zip(names, plan.fields())})
        plan.close()
    return fields
