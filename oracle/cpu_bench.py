"""CPU ORACLE timing — test/benchmark infrastructure only.

Times the oracle's NumPy restatement of the reference hot path (the same
DGEMM/ufunc sequence the reference executes) on this host's cores, for
bench.py's ``cpu_baseline`` and ``--impl reference`` legs.  The reference
itself (pure Python) cannot travel to the GPU box; the oracle is pinned to
it bit-for-bit on operands and to <= 1e-13 on trajectories
(tests/test_oracle_golden.py).

Ensemble (config 5): P worker processes x 1 BLAS thread, one member each,
started together behind a barrier; configs 1-4: one process
with all BLAS threads.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time


def _worker(idx, runs, dims, cmd_q, res_q, barrier):
    import numpy as np  # BLAS thread count comes from the env set by the parent

    from . import configs as ocfg
    from . import curvi_oracle as orc

    system = ocfg.config5_member(idx, dims, runs)
    tau = 1e-3
    ops = {c.name: orc.operands(c, tau) for c in system.comps}
    states = {c.name: np.array(c.initial) for c in system.comps}

    def advance(n):
        nonlocal states
        for _ in range(n):
            g = orc.react(system, states)
            states = {c.name: orc.split_step(ops[c.name], states[c.name], g[c.name]) for c in system.comps}

    advance(5)  # first-touch warm-up
    res_q.put(("ready", idx, 0.0))
    while True:
        n = cmd_q.get()
        if n is None:
            break
        barrier.wait()
        t0 = time.perf_counter()
        advance(n)
        res_q.put(("done", idx, time.perf_counter() - t0))


class CpuEnsemble:
    """Persistent pool of P oracle workers, one ensemble member each."""

    def __init__(self, workers: int, dims=(128, 256), runs: int = 512):
        self.P = workers
        self.dims = dims
        self.dof = 2 * dims[0] * dims[1]
        saved = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")}
        for k in saved:
            os.environ[k] = "1"
        ctx = mp.get_context("spawn")
        self.barrier = ctx.Barrier(workers)
        self.res_q = ctx.Queue()
        self.cmd_qs = [ctx.Queue() for _ in range(workers)]
        members = [int(round(i * (runs - 1) / max(workers - 1, 1))) for i in range(workers)]
        self.procs = [ctx.Process(target=_worker, args=(m, runs, dims, q, self.res_q, self.barrier), daemon=True)
                      for m, q in zip(members, self.cmd_qs)]
        for p in self.procs:
            p.start()
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        for _ in range(workers):
            self.res_q.get(timeout=600)

    def sample(self, steps: int) -> float:
        """Advance every worker's member by `steps`; returns the slowest
        worker's wall time (they start together)."""
        for q in self.cmd_qs:
            q.put(steps)
        return max(self.res_q.get(timeout=600)[2] for _ in range(self.P))

    def close(self):
        for q in self.cmd_qs:
            q.put(None)
        for p in self.procs:
            p.join(timeout=30)


def time_config(k: int, steps: int, warmup: int = 3, initial=None):
    """Seconds per step of the oracle on BASELINE config k (all BLAS threads)."""
    import numpy as np

    from . import configs as ocfg
    from . import curvi_oracle as orc

    system = ocfg.BUILDERS[k](initial=initial)
    m, t_star = ocfg.CONFIG_STEPS[k]
    tau = t_star / m
    ops = {c.name: orc.operands(c, tau) for c in system.comps}
    states = {c.name: np.array(c.initial) for c in system.comps}

    def advance(n):
        nonlocal states
        for _ in range(n):
            g = orc.react(system, states)
            states = {c.name: orc.split_step(ops[c.name], states[c.name], g[c.name]) for c in system.comps}

    advance(warmup)
    t0 = time.perf_counter()
    advance(steps)
    return (time.perf_counter() - t0) / steps
