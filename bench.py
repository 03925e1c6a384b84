#!/usr/bin/env python
"""Benchmark: BASELINE.json's metric (DOF*steps/s of fp64 split exponential
Euler) on its ensemble workload, config 5: 512 independent anomalous-disk
Schnakenberg runs (128 x 256 grid, 2 species, tau = 1e-3).

A bench "step" is one pass of the hot path over the batch: the whole
ensemble integrated over `--chunk` time steps (default the config's m =
1000), i.e. 512 * 2 * 128 * 256 DOF * 1000 time steps.  Runs are sharded
over ranks (strong scaling: the 512 runs are fixed); one NCCL gather of the
final fields to rank 0 follows the timed loop.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--chunk S]
    python bench.py --impl reference ...   # oracle port of the reference on host cores

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

RUNS = 512
DIMS = (128, 256)
NCOMP = 2
TAU = 1e-3
M_CONFIG = 1000
FP64_PEAK_TFLOPS = 37.05  # profiles/r01_fp64_peak.txt: DMMA m8n8k4 probe, 1965 MHz, no throttle
FP64_PEAK_CLOCK_MHZ = 1965.0
METRIC = "DOF*steps/s (fp64 split exponential Euler)"
UNIT = "DOF*steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--chunk", type=int, default=M_CONFIG, help="time steps per bench step")
    ap.add_argument("--impl", choices=["engine", "reference"], default="engine")
    ap.add_argument("--no-extras", action="store_true", help="skip per-config / CPU baseline legs")
    ap.add_argument("--theta", choices=["fft", "gemm"], default="fft",
                    help="periodic-theta factor as the exact FFT propagator or as two DMMA mu-mode products")
    return ap.parse_args()


def dof_total():
    return RUNS * NCOMP * DIMS[0] * DIMS[1]


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sms, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sampled = len(out.strip().splitlines())
        if not sampled:
            # a timed region shorter than the sampler's start-up: one query right after it
            try:
                out = subprocess.run(self.proc.args[:-2], capture_output=True, text=True, timeout=20).stdout
            except Exception:
                out = ""
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                maxes.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sms:
            return None
        loaded = [s for s in sms if s > 500] or sms
        loaded.sort()
        return {"sm_mhz": loaded[len(loaded) // 2], "sm_max_mhz": max(maxes), "reasons": sorted(reasons),
                "samples": len(sms) if sampled else 0}


# ---------------------------------------------------------------------------
# engine arm
# ---------------------------------------------------------------------------


def _free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_ranks(args):
    """`bench.py --gpus N` started without a launcher: re-exec under torchrun
    with N local ranks (one process per GPU).  Refuses loudly when the box has
    fewer than N GPUs instead of silently timing one rank."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible CUDA devices, found {have}",
              file=sys.stderr, flush=True)
        sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def dist_setup(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} rank(s)")
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py: rank {rank} wants cuda:{local}, only {torch.cuda.device_count()} device(s)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def per_rank(values, world):
    """Every rank's list of floats, on every rank (rank order)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(values, dtype=torch.float64, device="cuda")
    if world == 1:
        return [t.tolist()]
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [o.tolist() for o in out]


def max_over_ranks(value, world):
    import torch
    import torch.distributed as dist

    if world == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def kernel_roofline(plan, state, reps=20):
    """Average launch duration of each kernel of one step (CUDA events on the
    launching stream) and its achieved rate vs the measured peak."""
    import torch

    out = torch.empty_like(state)
    stream = torch.cuda.current_stream()
    rows = []
    pk = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    for stage in plan.step_kernels():
        flops, nbytes = plan.stage_info(stage)
        for _ in range(3):
            plan.run_stage(stage, state, out)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            plan.run_stage(stage, state, out)
        e1.record(stream)
        e1.synchronize()
        sec = e0.elapsed_time(e1) / 1e3 / reps
        if flops:
            row = {"kernel": f"gemm_stage{stage}", "bound": "tensor", "achieved": flops / sec / 1e12,
                   "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "flops_per_launch": flops}
        else:
            name = {-1: "fbuild", -2: "fused_fbuild_theta_fft"}.get(stage, f"theta_fft_stage{stage}")
            row = {"kernel": name, "bound": "hbm", "achieved": nbytes / sec / 1e9, "peak": hbm,
                   "unit": "GB/s", "bytes_per_launch": nbytes}
        row["frac"] = row["achieved"] / row["peak"]
        row["ms_per_launch"] = sec * 1e3
        rows.append(row)
    step_ms = sum(r["ms_per_launch"] for r in rows)
    for r in rows:
        r["share_of_step"] = r["ms_per_launch"] / step_ms
    return rows


def theta_variants(ens, init_dev, chunk, stream):
    """One bench step of config 5 under each theta mode (same inputs, same
    timing rules) so both formulations are reported side by side."""
    import torch

    from paper_2604_11558_b200.ensemble import Ensemble

    out = {}
    for mode in ("fft", "gemm"):
        e = Ensemble.__new__(Ensemble)
        from paper_2604_11558_b200.ensemble import ensemble_plan

        plan = ensemble_plan(ens.plan_template, "schnakenberg", ens.plan_params, TAU, theta=mode)
        state = init_dev.clone()
        bad = torch.full(state.shape[:2], 2**31 - 1, dtype=torch.int32, device="cuda")
        plan.run(state, 0, 32, bad)  # warm-up (graph capture)
        state.copy_(init_dev)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        plan.run(state, 0, chunk, bad)
        e1.record(stream)
        e1.synchronize()
        sec = e0.elapsed_time(e1) / 1e3
        out[mode] = {"value": dof_total() * chunk / sec, "ms_per_time_step": sec / chunk * 1e3}
        plan.close()
        del state
        del e
    return out


def ncu_traffic(kernel_key, theta):
    """Per-launch DRAM bytes (read + write) of a kernel from the committed ncu
    capture of one config-5 step (profiles/ncu_traffic.json), or None."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        return json.loads(p.read_text()).get(f"{theta}:{kernel_key}")
    except Exception:
        return None


def per_config_gpu(k, steps=200, warmup=20, theta=None):
    """One-GPU throughput of BASELINE config k (steps/s, DOF*steps/s) and the
    GEMM chain's FP64 fraction."""
    import numpy as np
    import torch

    from paper_2604_11558_b200 import configs
    from paper_2604_11558_b200.integrators import INT32_MAX, SplitPlan, prepare

    system = configs.BUILDERS[k]()
    m, t_star = configs.STEPS[k]
    tau = t_star / m
    geos = [prepare(c.ops, tau) for c in system.components]
    plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :], theta=theta)
    init = torch.from_numpy(np.stack([c.initial for c in system.components])[None]).cuda()
    state = init.clone()
    bad = torch.full((1, 2), INT32_MAX, dtype=torch.int32, device="cuda")
    plan.run(state, 0, warmup, bad)
    state.copy_(init)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.run(state, 0, steps, bad)
    e1.record()
    e1.synchronize()
    sec = e0.elapsed_time(e1) / 1e3 / steps
    dof = 2 * int(np.prod(system.components[0].ops.shape))
    flops = sum(plan.stage_info(s)[0] for s in range(plan.stage_count()))
    rows = kernel_roofline(plan, init, reps=10)
    gemm_sec = sum(r["ms_per_launch"] for r in rows if r["bound"] == "tensor") / 1e3
    return {"config": configs.NAMES[k], "theta": plan.theta, "dof": dof, "ms_per_step": sec * 1e3, "steps_per_s": 1.0 / sec,
            "dof_steps_per_s": dof / sec, "gemm_flops_per_step": flops,
            "gemm_chain_frac_fp64_peak": flops / gemm_sec / 1e12 / FP64_PEAK_TFLOPS,
            "step_frac_fp64_peak": flops / sec / 1e12 / FP64_PEAK_TFLOPS}


BULK_SURFACE = {
    # the paper's full-size bulk-surface runs (pkg/configs/ball_full.cfg, cylinder_full.cfg)
    "ball_full": ("bulk_surface_schnakenberg_ball", {"n_rho": 30, "n_theta": 50, "n_phi": 30}, 200000, 20.0),
    "cylinder_full": ("bsdib_cylinder", {"n_rho": 160, "n_theta": 160, "n_z": 20}, 8000, 50.0),
}


def bulk_surface_gpu(key, steps=320, warmup=32):
    """One-GPU throughput of a full-size bulk-surface model: one coupled step
    = coupling kernel + bulk step_split + surface step_split (cg_coupled_run,
    graph-replayed)."""
    import numpy as np
    import torch

    from paper_2604_11558_b200 import models
    from paper_2604_11558_b200.coupled import CoupledPlan
    from paper_2604_11558_b200.integrators import prepare

    name, dims, m, t_star = BULK_SURFACE[key]
    system = models.build_system(name, dims, 1)
    tau = t_star / m
    comps = system.components
    plan = CoupledPlan([prepare(c.ops, tau) for c in comps], system.kinetics, lifts=[c.lift for c in comps])
    plan.load([c.initial for c in comps])
    plan.run(0, warmup)
    plan.load([c.initial for c in comps])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.run(0, steps)
    e1.record()
    e1.synchronize()
    sec = e0.elapsed_time(e1) / 1e3 / steps
    dof = sum(int(np.prod(c.ops.shape)) for c in comps)
    ok = bool((plan.first_bad.cpu().numpy() == 2**31 - 1).all())
    plan.close()
    return {"model": name, "dims": dims, "dof": dof, "ms_per_step": sec * 1e3, "dof_steps_per_s": dof / sec,
            "paper_run_s": sec * m, "paper_steps": m, "no_divergence": ok}


def bulk_surface_cpu(key, steps=3):
    """The same coupled step on the host: the real reference (baseline/_ref)
    through its own run_simulation when installed, else the oracle port."""
    import time

    from oracle import ref_bench

    name, dims, m, t_star = BULK_SURFACE[key]
    tau = t_star / m
    threads = os.environ.get("OPENBLAS_NUM_THREADS", "default (all cores)")
    if ref_bench.available():
        from oracle import ref_configs

        ref_configs.load_curvipat()
        from curvipat import models as ref_models

        system = ref_models.build_system(name, dims, 1)
        sec = ref_bench.timed_run(system, 1, steps, tau) / steps
        dof = sum(int(c.initial.size) for c in system.components)
        return {"model": name, "ms_per_step": sec * 1e3, "dof_steps_per_s": dof / sec, "kind": "reference",
                "threads": threads}
    from oracle import configs as ocfg
    from oracle import curvi_oracle as orc
    from paper_2604_11558_b200 import models

    system = models.build_system(name, dims, 1)
    init = [c.initial for c in system.components]
    d = tuple(dims.values())
    osys = ocfg.bs_ball(d, initial=init) if key.startswith("ball") else ocfg.bs_cylinder(d, initial=init)
    orc.integrate(osys, 1, tau)
    t0 = time.perf_counter()
    orc.integrate(osys, steps, steps * tau)
    sec = (time.perf_counter() - t0) / steps
    dof = sum(int(c.initial.size) for c in system.components)
    return {"model": name, "ms_per_step": sec * 1e3, "dof_steps_per_s": dof / sec, "kind": "port",
            "threads": threads}


def engine_arm(args):
    import numpy as np
    import torch

    from paper_2604_11558_b200 import configs
    from paper_2604_11558_b200.ensemble import Ensemble, gather_fields, shard_range

    from paper_2604_11558_b200 import integrators

    integrators.THETA_MODE = args.theta
    world, rank, local = dist_setup(args)
    lo, hi = shard_range(RUNS, rank, world)
    inputs = configs.config5_inputs(lo, hi - lo)
    params = np.stack([[g, 0.1, 0.9] for g in inputs.gammas])
    ens = Ensemble(inputs.template, "schnakenberg", params, TAU)
    ens.load(inputs.states)
    init_dev = ens.host_in.to("cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # 256 MB > 126 MB L2
    stream = torch.cuda.current_stream()
    chunk = args.chunk

    def one_device_step(timed):
        ens.state.copy_(init_dev)
        ens.first_bad.fill_(2**31 - 1)
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ens.plan.run(ens.state, 0, chunk, ens.first_bad)
        e1.record(stream)
        return e0, e1

    for _ in range(args.warmup):
        one_device_step(False)
    barrier(world)
    clocks = ClockSampler(local) if rank == 0 else None
    events = [one_device_step(True) for _ in range(args.steps)]
    barrier(world)
    cl = clocks.stop() if clocks else None
    dev_sec = sum(a.elapsed_time(b) for a, b in events) / 1e3
    dev_sec = max_over_ranks(dev_sec, world)
    bad = ens.first_bad.cpu().numpy()

    # end to end through the public Ensemble API: pinned host -> device, step, device -> host
    for _ in range(max(1, args.warmup)):
        ens.advance(chunk)
    barrier(world)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        ens.advance(chunk, from_host=True, to_host=True)
    e1.record(stream)
    barrier(world)
    e2e_local = e0.elapsed_time(e1) / 1e3
    e2e_sec = max_over_ranks(e2e_local, world)
    dev_local = sum(a.elapsed_time(b) for a, b in events) / 1e3
    ranks = per_rank([float(lo), float(hi), dev_local, e2e_local], world)

    # the ensemble's one collective: final physical fields to rank 0
    t0 = time.perf_counter()
    lifts = torch.tensor([1.0, 0.9], dtype=torch.float64, device="cuda").view(1, 2, 1, 1)
    phys = ens.state + lifts
    if world > 1:
        gathered = gather_fields(phys, RUNS)
    else:
        gathered = phys
    barrier(world)
    gather_ms = (time.perf_counter() - t0) * 1e3
    finite = bool(torch.isfinite(gathered).all().item()) if rank == 0 else True

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    total_dofsteps = dof_total() * chunk * args.steps
    value = total_dofsteps / dev_sec
    e2e_value = total_dofsteps / e2e_sec
    rows = kernel_roofline(ens.plan, init_dev)
    dom = max((r for r in rows), key=lambda r: r["share_of_step"])
    gemm_flops = sum(ens.plan.stage_info(s)[0] for s in range(ens.plan.stage_count()))
    # kernels one time step launches (fused front + GEMM in fft mode; launch list:
    # profiles/r01_v10_launches_summary.txt) x time steps, + the step-counter reset per cg_run
    # with lanes every lane launches its own kernels (and its own step-counter reset)
    lanes = ens.plan.lanes
    launches_per_step = lanes * (chunk * len(ens.plan.step_kernels()) + 1)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev_sec / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: reference-seeded xoshiro256++ initial fields (seed 1+i), gamma_i swept over [50, 200]",
        "config": {
            "workload": "BASELINE config 5: ensemble of 512 anomalous-disk Schnakenberg runs, 128x256 grid, "
                        "2 species, tau=1e-3; bench step = whole ensemble over `time_steps_per_bench_step`",
            "runs": RUNS, "grid": list(DIMS), "species": NCOMP, "tau": TAU,
            "time_steps_per_bench_step": chunk, "dof": dof_total(),
            "theta": args.theta + (" (exact real-FFT propagator for Q diag(Phi) Q^T)" if args.theta == "fft"
                                   else " (two DMMA mu-mode products, the reference's factorisation)"),
            "parallelism": f"ensemble shards over {world} GPU(s), no data-path collective",
            "lanes": lanes,
            "l2": "state 268 MB/GPU at N=1 exceeds 126 MB L2; 256 MB L2 flush between timed bench steps",
        },
        "steps_per_s": chunk * args.steps / dev_sec,
        # whole-step FP64 fraction: dense phi/eigenbasis flops of all runs / time / (peak x GPUs)
        "fp64_frac_of_peak_step": gemm_flops / (hi - lo) * RUNS * chunk * args.steps / dev_sec / 1e12
        / (FP64_PEAK_TFLOPS * world),
        "roofline": {"bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"], "unit": dom["unit"],
                     "frac": dom["frac"], "traffic": ncu_traffic(dom["kernel"], args.theta), "kernel": dom["kernel"],
                     "peak_source": ("measured DMMA peak, profiles/r01_fp64_peak.txt (MEASURED_PEAKS.json has "
                                     "no fp64 figure)") if dom["bound"] == "tensor" else "MEASURED_PEAKS.json hbm_gbs"},
        "kernels": rows,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": ens.nbytes, "d2h_bytes_per_step": ens.nbytes,
                "api": "paper_2604_11558_b200.ensemble.Ensemble.advance (pinned host in/out)"},
        "gpu_launches": launches_per_step * args.steps,
        "gather_ms": gather_ms,
        "per_rank": [{"rank": r, "runs": [int(v[0]), int(v[1])], "device_s": v[2], "e2e_s": v[3],
                      "value": (v[1] - v[0]) * NCOMP * DIMS[0] * DIMS[1] * chunk * args.steps / v[2]}
                     for r, v in enumerate(ranks)],
        "diverged_runs": int((bad.min(axis=1) < 2**31 - 1).sum()),
        "finite": finite,
    }
    if cl:
        line["clocks"] = cl
        if line["roofline"]["bound"] == "tensor" and cl.get("sm_mhz"):
            # the FP64 peak was measured at the maximum SM clock; the timed region runs under the
            # box's power cap: state both clocks and the fraction against the clock-scaled peak
            rf = line["roofline"]
            rf["peak_clock_mhz"] = FP64_PEAK_CLOCK_MHZ
            rf["run_clock_mhz"] = cl["sm_mhz"]
            rf["frac_at_run_clock"] = rf["achieved"] / (rf["peak"] * cl["sm_mhz"] / FP64_PEAK_CLOCK_MHZ)
    if world == 1 and not args.no_extras:
        line["cpu_baseline"] = cpu_baseline_ensemble(sample_steps=200)
        line["per_config"] = [per_config_gpu(k, theta=t) for k in (1, 2, 3, 4) for t in ("fft", "gemm")]
        line["variants"] = theta_variants(ens, init_dev, chunk, stream)
        line["per_config_cpu"] = cpu_per_config()
        line["bulk_surface"] = [bulk_surface_gpu(k) for k in BULK_SURFACE]
        line["bulk_surface_cpu"] = [bulk_surface_cpu(k) for k in BULK_SURFACE]
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU legs (oracle port of the reference)
# ---------------------------------------------------------------------------


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _cpu_pool(P):
    """P host workers, one config-5 member each: the real reference from
    baseline/_ref when installed (kind "reference"), else the oracle port."""
    from oracle import ref_bench

    if ref_bench.available():
        return ref_bench.RefEnsemble(P, DIMS, RUNS), "reference"
    from oracle.cpu_bench import CpuEnsemble

    return CpuEnsemble(P, DIMS, RUNS), "port"


def _host_facts():
    from oracle import ref_bench

    return {"cpu_model": ref_bench.cpu_model(), "host_cores": host_cores()}


def cpu_baseline_ensemble(sample_steps=200, workers=None):
    """SURVEY 8(d) steps 1-3 on the GPU box's host: all cores (one process
    per core x 1 BLAS thread, one member each) and the P = 1 leg, the CPU
    model, the BLAS build, and setup (build_system + IC, prepare) reported
    apart from stepping."""
    P = workers or host_cores()
    pool, kind = _cpu_pool(P)
    try:
        sec = pool.sample(sample_steps)
        setup = getattr(pool, "setup", None)
        blas = getattr(pool, "blas", None)
    finally:
        pool.close()
    one, _ = _cpu_pool(1)
    try:
        sec1 = one.sample(sample_steps)
    finally:
        one.close()
    dof = NCOMP * DIMS[0] * DIMS[1]
    what = ("curvipat.integrators.run_simulation from baseline/_ref (the unmodified reference), stepping timed "
            "by its own sample_hook" if kind == "reference" else
            "oracle/ NumPy restatement of curvipat's split EE step (baseline/_ref not installed)")
    return {"value": P * dof * sample_steps / sec, "unit": UNIT, "cores": P, "kind": kind,
            "sample": f"{P} ensemble members x {sample_steps} steps, one process per core, 1 BLAS thread each "
                      f"({what}; {sec:.2f} s wall)",
            "p1": {"value": dof * sample_steps / sec1, "cores": 1, "ms_per_step": sec1 / sample_steps * 1e3},
            "setup_s": setup, "blas": blas, **_host_facts()}


def cpu_per_config():
    """Configs 1-4 on the host at 1 BLAS thread and at all cores (one
    process), through the real reference when installed."""
    from threadpoolctl import threadpool_limits

    from oracle import ref_bench

    out = []
    for k, steps in ((1, 100), (2, 10), (3, 3), (4, 3)):
        dims = {1: (64, 128), 2: (512, 256), 3: (64, 128, 128), 4: (100, 100, 100)}[k]
        dof = 2
        for d in dims:
            dof *= d
        row = {"config": k}
        for label, limit in (("p1", 1), ("pall", None)):
            with threadpool_limits(limits=limit):
                if ref_bench.available():
                    r = ref_bench.time_config(k, steps)
                    sec, kind = r["sec_per_step"], "reference"
                    row["setup_s"] = {"build_system_ic_s": r["build_system_ic_s"], "prepare_s": r["prepare_s"]}
                else:
                    from oracle.cpu_bench import time_config

                    sec, kind = time_config(k, steps), "port"
            row[label] = {"ms_per_step": sec * 1e3, "dof_steps_per_s": dof / sec,
                          "threads": 1 if limit == 1 else host_cores()}
            row["kind"] = kind
        out.append(row)
    return out


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    P = host_cores()
    per_step = 20  # time steps each member advances per bench step (bounded sample)
    pool, kind = _cpu_pool(P)
    try:
        for _ in range(args.warmup):
            pool.sample(per_step)
        total = 0.0
        for _ in range(args.steps):
            total += pool.sample(per_step)
        setup = getattr(pool, "setup", None)
    finally:
        pool.close()
    dof = NCOMP * DIMS[0] * DIMS[1]
    value = P * dof * per_step * args.steps / total
    what = ("the unmodified reference curvipat (baseline/_ref) through curvipat.integrators.run_simulation, "
            "stepping timed by its own sample_hook" if kind == "reference" else
            "oracle/ NumPy port of curvipat's split EE (baseline/_ref not installed)")
    sample = (f"{P} of the 512 ensemble members x {per_step} time steps per bench step, one process per core "
              f"x 1 BLAS thread ({what})")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": "synthetic: reference-seeded xoshiro256++ initial fields",
        "config": {"workload": "BASELINE config 5 ensemble (512 x anomalous disk 128x256), bounded CPU sample",
                   "runs_sampled": P, "time_steps_per_bench_step": per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": P, "kind": kind, "sample": sample,
                         "setup_s": setup, **_host_facts()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if args.impl == "engine" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        launch_ranks(args)
    if args.impl == "reference":
        reference_arm(args)
    else:
        engine_arm(args)


if __name__ == "__main__":
    main()
