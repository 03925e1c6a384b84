"""CPU REFERENCE timing -- benchmark infrastructure only, never product code.

Times the REAL reference (curvipat, pip-installed into the git-ignored
``baseline/_ref`` with ``pip install --no-index --no-build-isolation
--no-deps --target baseline/_ref <copy of /root/reference/pkg>``) through its
own public API on this host's cores, for bench.py's ``--impl reference`` arm
and ``cpu_baseline`` (SURVEY 8(d) "CPU baseline timing"):

- the stepping time is taken INSIDE ``curvipat.integrators.run_simulation``
  by its own ``sample_hook`` (perf_counter at the end of warm-up step W and
  of step W+n), so prepare, IC and build_system are excluded and reported
  separately, and the stock loop (kinetics closure, step_split per
  component, divergence guard) is what is timed;
- ensemble (config 5): P worker processes x 1 BLAS thread, one member each,
  released together by a barrier; aggregate DOF*steps/s = P * DOF * n /
  slowest worker's time;
- single configs 1-4: one process, BLAS threads as given.

When baseline/_ref is absent the caller falls back to oracle/cpu_bench.py
(the NumPy port) and says so in ``kind``.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import platform
import time

from .ref_configs import REF_DIR

TAU5 = 1e-3


def available() -> bool:
    return (REF_DIR / "curvipat" / "__init__.py").exists()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def blas_info() -> list:
    """threadpoolctl's view of the BLAS numpy links (name, version, threads)."""
    try:
        import numpy  # noqa: F401
        from threadpoolctl import threadpool_info

        return [{k: d.get(k) for k in ("internal_api", "version", "num_threads", "threading_layer")}
                for d in threadpool_info() if d.get("user_api") == "blas"]
    except Exception as exc:  # noqa: BLE001
        return [{"error": str(exc)}]


def timed_run(system, warm: int, n: int, tau: float) -> float:
    """Seconds for steps warm+1 .. warm+n of the reference's own
    run_simulation (its sample_hook fires after step `warm` and after the
    last step)."""
    from curvipat.integrators import run_simulation

    marks = {}

    def hook(step, t, states):
        marks[step] = time.perf_counter()

    run_simulation(system, warm + n, (warm + n) * tau, record_every=warm, sample_hook=hook)
    return marks[warm + n] - marks[warm]


def _setup_times(build, tau):
    """(build_system + IC seconds, prepare seconds) of one system."""
    from curvipat.integrators import prepare

    t0 = time.perf_counter()
    system = build()
    t1 = time.perf_counter()
    for c in system.components:
        prepare(c.ops, tau)
    t2 = time.perf_counter()
    return system, t1 - t0, t2 - t1


def _worker(idx, runs, dims, cmd_q, res_q, barrier):
    from . import ref_configs

    ref_configs.load_curvipat()
    system, t_build, t_prep = _setup_times(lambda: ref_configs.ref_member(idx, dims, runs), TAU5)
    timed_run(system, 2, 3, TAU5)  # first-touch warm-up
    res_q.put(("ready", idx, {"build_s": t_build, "prepare_s": t_prep, "blas": blas_info()}))
    while True:
        n = cmd_q.get()
        if n is None:
            break
        barrier.wait()
        res_q.put(("done", idx, timed_run(system, 5, n, TAU5)))


class RefEnsemble:
    """P reference worker processes (1 BLAS thread each), one config-5
    member each, members spread over the 512-run sweep."""

    def __init__(self, workers: int, dims=(128, 256), runs: int = 512):
        self.P = workers
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
        ready = [self.res_q.get(timeout=900) for _ in range(workers)]
        infos = [r[2] for r in ready]
        self.setup = {"build_system_ic_s": max(i["build_s"] for i in infos),
                      "prepare_s": max(i["prepare_s"] for i in infos)}
        self.blas = infos[0]["blas"]

    def sample(self, steps: int) -> float:
        """Advance every worker's member by `steps` timed steps; the slowest
        worker's seconds (they start together)."""
        for q in self.cmd_qs:
            q.put(steps)
        return max(self.res_q.get(timeout=900)[2] for _ in range(self.P))

    def close(self):
        for q in self.cmd_qs:
            q.put(None)
        for p in self.procs:
            p.join(timeout=30)


def time_config(k: int, steps: int, warm: int = 2) -> dict:
    """Reference seconds per step of BASELINE config k (this process's BLAS
    threads) plus its setup times."""
    from . import ref_configs

    ref_configs.load_curvipat()
    m, t_star = ref_configs.STEPS[k]
    tau = t_star / m
    system, t_build, t_prep = _setup_times(lambda: ref_configs.ref_config(k, ref_configs.FULL[k]), tau)
    sec = timed_run(system, warm, steps, tau) / steps
    return {"sec_per_step": sec, "build_system_ic_s": t_build, "prepare_s": t_prep}
