"""Ensembles of independent runs (seed / parameter sweeps), batched into one
plan per GPU and sharded over ranks.

The reference has no parallel path; its docs call runs "embarrassingly
parallel".  Here rank r of G takes the contiguous runs
[r R / G, (r+1) R / G); runs never communicate while stepping, and one
collective at the end gathers the final physical fields to rank 0 (NCCL over
NVLink on GPUs; gloo in the CPU tests of the gather logic).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .integrators import INT32_MAX, DivergenceError, SplitPlan, engine_kinetics, prepare


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) of `total` runs owned by `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (rank * total) // world, ((rank + 1) * total) // world


def gather_fields(local, total: int, group=None, dst: int = 0):
    """Gather per-rank blocks [n_r, ...] of a [total, ...] array to `dst`.

    Uses torch.distributed.gather on equal-size padded blocks (NCCL needs
    equal shapes); returns the [total, ...] tensor on dst and None elsewhere.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    biggest = max(shard_range(total, r, world)[1] - shard_range(total, r, world)[0] for r in range(world))
    # gloo moves host tensors only: stage device blocks through host memory
    dev = _comm_device(local.device, group)
    pad = torch.zeros((biggest,) + tuple(local.shape[1:]), dtype=local.dtype, device=dev)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    parts = []
    for r in range(world):
        lo, hi = shard_range(total, r, world)
        parts.append(bufs[r][: hi - lo])
    return torch.cat(parts, dim=0).to(local.device)


def _comm_device(want, group=None):
    """Device a collective's tensors must live on: the tensor's own for NCCL,
    the host for gloo."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return want if want.type == "cuda" else torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def agree(value: int, op: str, group=None) -> int:
    """All-reduce one integer over the group (``op`` "min" or "max"); the
    value itself when no process group is initialised.  Ranks use it to reach
    the same decision (raise / continue) before any later collective, so a
    rank-local error can never leave the others blocked in a gather."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return int(value)
    t = torch.tensor([int(value)], dtype=torch.int64, device=_comm_device(torch.device("cpu"), group))
    dist.all_reduce(t, op=dist.ReduceOp.MIN if op == "min" else dist.ReduceOp.MAX, group=group)
    return int(t.item())


def ensemble_plan(template, kin_kind: str, params: np.ndarray, tau: float, theta: str | None = None) -> SplitPlan:
    """One batched plan: operators from the template system, per-run kinetics
    parameters ``params`` [B, P]."""
    geos = [prepare(c.ops, tau) for c in template.components]
    lifts = [float(getattr(c, "lift", 0.0)) for c in template.components]
    return SplitPlan(geos, batch=params.shape[0], kinetics=kin_kind, kin_params=params, lifts=lifts, theta=theta)


def _check_shared(systems) -> bool:
    """True when every member shares the first member's operators (one
    operator set per component); False for a heterogeneous ensemble (per-run
    operator sets: coefficients or domain sizes differ, grids agree).  Names,
    lifts and the kinetics kind must always agree."""
    ref = systems[0]
    shared = True
    shape = [tuple(c.ops.shape) for c in ref.components]
    for s in systems[1:]:
        if [c.name for c in s.components] != [c.name for c in ref.components]:
            raise NotImplementedError("ensemble members must have the same components")
        if [tuple(c.ops.shape) for c in s.components] != shape:
            raise NotImplementedError("ensemble members must share grid extents")
        for a, b in zip(ref.components, s.components):
            if a.lift != b.lift:
                raise NotImplementedError("ensemble members must share lifts")
            if a.ops is not b.ops and not _same_ops(a.ops, b.ops):
                shared = False
        if engine_kinetics(s).kind != engine_kinetics(ref).kind:
            raise NotImplementedError("ensemble members must share the kinetics kind")
    return shared


def _same_ops(x, y) -> bool:
    if x.coeff != y.coeff or str(x.geometry) != str(y.geometry):
        return False
    for axis in ("rho", "theta", "phi", "z"):
        p, q = getattr(x, axis), getattr(y, axis)
        if (p is None) != (q is None):
            return False
        if p is None:
            continue
        for attr in ("a", "b", "c", "grid", "diag", "off"):
            u, v = getattr(p, attr, None), getattr(q, attr, None)
            if not np.array_equal(np.asarray(u), np.asarray(v)):
                return False
    wx, wy = getattr(x, "rho_weights", None), getattr(y, "rho_weights", None)
    if (wx is None) != (wy is None):
        return False
    return wx is None or np.array_equal(wx.values, wy.values)


class Ensemble:
    """A persistent batched engine for B runs that share operators: the plan,
    device state and pinned host staging buffers are allocated once, so each
    :meth:`advance` is H2D + graph-replayed stepping + D2H on one stream.

    ``params`` [B, P] are the per-run kinetics parameters, ``lifts`` per
    component.  This is the call bench.py times for its end-to-end number.
    """

    def __init__(self, template, kin_kind: str, params, tau: float):
        import torch

        self.plan_template = template
        self.plan_params = np.asarray(params, dtype=np.float64)
        self.plan = ensemble_plan(template, kin_kind, self.plan_params, tau)
        self.tau = tau
        shape = self.plan.state_shape
        self.state = torch.empty(shape, dtype=torch.float64, device="cuda")
        self.first_bad = torch.full(shape[:2], INT32_MAX, dtype=torch.int32, device="cuda")
        self.host_in = torch.empty(shape, dtype=torch.float64, pin_memory=True)
        self.host_out = torch.empty(shape, dtype=torch.float64, pin_memory=True)
        self.step = 0
        # host_in may be rewritten only after the last upload has read it;
        # host_out is valid once `downloaded` has completed
        self.uploaded = torch.cuda.Event()
        self.downloaded = torch.cuda.Event()

    @property
    def nbytes(self) -> int:
        return self.state.numel() * 8

    def load(self, host_states) -> None:
        """Copy numpy/torch host states into the pinned buffer (outside any
        timing).  Waits for the previous :meth:`advance`'s upload to have read
        the buffer first, so a pending asynchronous copy never sees new data."""
        import torch

        self.uploaded.synchronize()
        self.host_in.copy_(torch.as_tensor(np.ascontiguousarray(host_states)))

    def advance(self, nsteps: int, *, from_host: bool = True, to_host: bool = True, blocking: bool = True):
        """Optionally upload host_in, step nsteps, optionally download to host_out.

        With a laned plan every lane uploads, steps and downloads its own run
        block on its own stream, so lane 1's upload runs under lane 0's
        stepping and lane 0's download under lane 1's tail.

        Returns ``host_out``.  With ``blocking`` (default) the call returns
        once the download has landed, so the buffer can be read at once; with
        ``blocking=False`` it returns immediately and ``self.downloaded`` (a
        CUDA event on the caller's stream) marks when host_out is valid."""
        import torch

        if from_host:
            self.first_bad.fill_(INT32_MAX)
        lanes = self.plan.lane_blocks()
        if not lanes:
            if from_host:
                self.state.copy_(self.host_in, non_blocking=True)
            self.plan.run(self.state, 0 if from_host else self.step, nsteps, self.first_bad)
        else:
            cur = torch.cuda.current_stream()
            ready = torch.cuda.Event()
            ready.record(cur)
            for lo, hi, sub, stream in lanes:
                stream.wait_event(ready)
                with torch.cuda.stream(stream):
                    if from_host:
                        self.state[lo:hi].copy_(self.host_in[lo:hi], non_blocking=True)
                    sub.run(self.state[lo:hi], 0 if from_host else self.step, nsteps, self.first_bad[lo:hi])
                    if to_host:
                        self.host_out[lo:hi].copy_(self.state[lo:hi], non_blocking=True)
            for _, _, _, stream in lanes:
                cur.wait_stream(stream)
        if from_host:
            self.uploaded.record()
            self.step = 0
        self.step += nsteps
        if to_host and not lanes:
            self.host_out.copy_(self.state, non_blocking=True)
        self.downloaded.record()
        if to_host and blocking:
            self.downloaded.synchronize()
        return self.host_out


@dataclass
class EnsembleResult:
    fields: object  # [R, C, ...] physical fields on rank 0 (numpy or torch), None elsewhere
    first_bad: np.ndarray  # [n_local, C] first diverged step (INT32_MAX = never), this rank's runs
    start: int
    stop: int
    steps: int
    tau: float
    times: list | None = None  # sample times (record_every / diagnostics), else None
    series: object = None  # [R, C, nsamples] integral means on rank 0 (numpy or torch), None elsewhere


def run_ensemble(systems, m: int, t_star: float, *, group=None, gather: bool = True,
                 as_torch: bool = False, raise_on_divergence: bool = False,
                 record_every: int | None = None, diagnostics=None, setup: str = "host") -> EnsembleResult:
    """Advance every member of ``systems`` (a list of CoupledSystem on one
    grid) by m steps of tau = t*/m; shard over the torch.distributed group
    when one is initialised.  Members sharing their operators run on one
    operator set per component; members that differ (diffusion coefficients,
    domain sizes: a parameter sweep) get one prepared set per run.

    ``diagnostics`` (a ``models.MeanDiagnostics``, e.g.
    ``mean_diagnostics(systems[0])``) samples every member's integral means on
    the device at step 0, every ``record_every`` steps and at m, as
    run_simulation does for one run; the [R, C, nsamples] series is gathered
    with the fields.

    ``setup``: where a heterogeneous ensemble's per-run operator sets are
    prepared -- ``"host"`` (``prepare`` per run and component, the reference's
    path) or ``"device"`` (``device_setup.prepare_device``: every eigenproblem
    and phi1 table of the shard in batched GPU launches)."""
    import torch
    import torch.distributed as dist

    if m < 1:
        raise ValueError("need at least one time step")
    if t_star <= 0:
        raise ValueError("t_star must be positive")
    if setup not in ("host", "device"):
        raise ValueError(f"setup must be 'host' or 'device', got {setup!r}")
    R = len(systems)
    if R == 0:
        raise ValueError("empty ensemble")
    dist_on = dist.is_available() and dist.is_initialized()
    world = dist.get_world_size(group) if dist_on else 1
    rank = dist.get_rank(group) if dist_on else 0
    lo, hi = shard_range(R, rank, world)
    mine = systems[lo:hi]
    tau = t_star / m
    sample_steps = None
    if diagnostics is not None:
        from .models import MeanDiagnostics

        if not isinstance(diagnostics, MeanDiagnostics):
            raise NotImplementedError("ensemble diagnostics must be models.mean_diagnostics(...) (device-evaluated)")
        every = record_every or m
        sample_steps = [0]
        while sample_steps[-1] < m:
            sample_steps.append(min(m, (sample_steps[-1] // every + 1) * every))
    names = [c.name for c in systems[0].components]
    ncomp = len(names)
    # Setup can fail on one shard only (a member with other components, an
    # unsupported kinetics, a bad operator): every rank learns whether any
    # failed before it steps, so none is left waiting in the final gather.
    plan = None
    setup_error = None
    if mine:
        try:
            shared = _check_shared(mine)
            kin = engine_kinetics(mine[0])
            params = np.stack([engine_kinetics(s).param_vector() for s in mine])
            if shared:
                plan = ensemble_plan(mine[0], kin.kind, params, tau)
            else:
                # heterogeneous ensemble: one prepared operator set per (run, component)
                if setup == "device":
                    from .device_setup import prepare_device

                    geos = prepare_device([c.ops for s in mine for c in s.components], tau)
                else:
                    geos = [prepare(c.ops, tau) for s in mine for c in s.components]
                lifts = [float(getattr(c, "lift", 0.0)) for c in mine[0].components]
                plan = SplitPlan(geos, batch=len(mine), kinetics=kin.kind, kin_params=params, lifts=lifts,
                                 ops_per_run=True)
        except Exception as exc:  # re-raised below, after the ranks agree
            setup_error = exc
    failed_rank = agree(rank if setup_error is not None else world, "min", group)
    if failed_rank < world:
        if setup_error is not None:
            raise setup_error
        raise RuntimeError(f"run_ensemble: setup failed on rank {failed_rank}; see that rank's error")
    if mine:
        host = np.stack([np.stack([np.asarray(c.initial, dtype=np.float64) for c in s.components]) for s in mine])
        state = torch.from_numpy(np.ascontiguousarray(host)).to("cuda")
        first_bad = torch.full((hi - lo, plan.ncomp), INT32_MAX, dtype=torch.int32, device="cuda")
        if sample_steps is None:
            plan.run(state, 0, m, first_bad)
        else:
            means = diagnostics.device_means(names, hi - lo)
            series = torch.empty((len(sample_steps), hi - lo, ncomp), dtype=torch.float64, device="cuda")
            means.into(state, series[0])
            for i in range(1, len(sample_steps)):
                plan.run(state, sample_steps[i - 1], sample_steps[i] - sample_steps[i - 1], first_bad)
                means.into(state, series[i])
            series = series.permute(1, 2, 0).contiguous()
        lifts = torch.tensor([float(getattr(c, "lift", 0.0)) for c in mine[0].components],
                             dtype=torch.float64, device="cuda")
        phys = state + lifts.view((1, -1) + (1,) * (state.dim() - 2))
        bad = first_bad.cpu().numpy()
    else:
        shape = tuple(systems[0].components[0].ops.shape)
        phys = torch.zeros((0, len(systems[0].components)) + shape, dtype=torch.float64, device="cuda")
        bad = np.zeros((0, len(systems[0].components)), dtype=np.int32)
        if sample_steps is not None:
            series = torch.zeros((0, ncomp, len(sample_steps)), dtype=torch.float64, device="cuda")
    if raise_on_divergence:
        # the first bad step over ALL ranks' runs, raised by every rank together
        s = agree(int(bad.min()) if bad.size else INT32_MAX, "min", group)
        if s < INT32_MAX:
            raise DivergenceError(f"ensemble run diverged at step {s}", step=s)
    if dist_on and gather and world > 1:
        full = gather_fields(phys, R, group=group)
    else:
        full = phys if rank == 0 else None
    if full is not None and not as_torch:
        full = full.cpu().numpy()
    times = full_series = None
    if sample_steps is not None:
        times = [k * tau for k in sample_steps]
        if dist_on and gather and world > 1:
            full_series = gather_fields(series, R, group=group)
        else:
            full_series = series if rank == 0 else None
        if full_series is not None and not as_torch:
            full_series = full_series.cpu().numpy()
    return EnsembleResult(full, bad, lo, hi, m, tau, times, full_series)
