"""GPU parity: the CUDA path (through libcurvigpu's C ABI) against the
reference's golden fixtures and the CPU oracle on identical seeded inputs.

Tolerance (north_star): relative inf-norm on physical fields <= 1e-10 after
1 step and <= 1e-8 after 100 steps.  Single operations (diffusion action,
one split step on random data) are held to 1e-12.
"""

import numpy as np
import pytest

from oracle import configs as ocfg
from oracle import curvi_oracle as orc
from paper_2604_11558_b200 import configs as pcfg
from paper_2604_11558_b200.integrators import (
    INT32_MAX,
    DivergenceError,
    SplitPlan,
    apply_diffusion,
    prepare,
    run_simulation,
    step_split,
)

from ._cases import CASES, engine_base
from .conftest import rel_inf

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["gemm", "fft"])
def theta_mode(request, monkeypatch):
    """Every parity case runs with the theta factor as two DMMA mu-mode
    products (the reference's formulation) and as the FFT propagator."""
    from paper_2604_11558_b200 import integrators

    monkeypatch.setattr(integrators, "THETA_MODE", request.param)
    return request.param

SMALL = {1: (16, 32), 2: (24, 16), 3: (8, 16, 16), 4: (10, 12, 10), 5: (16, 32)}
STEP1_TOL = 1e-10
STEP100_TOL = 1e-8


@pytest.mark.parametrize("name", CASES)
def test_apply_diffusion_matches_reference(golden, name):
    base = engine_base(name)
    for tau in (0.037, 0.0):
        key = f"{name}_tau{tau}"
        out = apply_diffusion(prepare(base, tau), golden.steps[key + "_W"])
        assert rel_inf(out, golden.steps[key + "_MW"]) <= 1e-12


@pytest.mark.parametrize("name", CASES)
def test_step_split_matches_reference(golden, name):
    base = engine_base(name)
    for tau in (0.037, 0.0):
        key = f"{name}_tau{tau}"
        W, G = golden.steps[key + "_W"], golden.steps[key + "_G"]
        out = step_split(prepare(base, tau), W, G)
        if tau == 0.0:
            assert np.array_equal(out, W)  # reference tests/test_integrators.py:116-123
        assert rel_inf(out, golden.steps[key + "_out"]) <= 1e-12


def test_step_split_torch_in_torch_out(golden):
    import torch

    key = "disk_20x36_tau0.037"
    W = torch.from_numpy(golden.steps[key + "_W"]).cuda()
    G = torch.from_numpy(golden.steps[key + "_G"]).cuda()
    out = step_split(prepare(engine_base("disk_20x36"), 0.037), W, G)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    assert rel_inf(out.cpu().numpy(), golden.steps[key + "_out"]) <= 1e-12


@pytest.mark.parametrize("name", ["disk_20x36", "sphere_40x34", "ball_12x10x18", "cylinder_9x20x24"])
def test_constants_are_fixed_points(name):
    base = engine_base(name)
    ops = prepare(base, 0.05)
    W = np.full(base.shape, 3.7)
    out = step_split(ops, W, np.zeros(base.shape))
    if name.startswith("cylinder_9"):  # Neumann-Neumann z: constants are fixed too
        assert np.max(np.abs(out - W)) <= 1e-10
    else:
        assert np.max(np.abs(out - W)) <= 1e-10


def test_zero_field_is_fixed_bitwise_cylinder_dirichlet():
    base = engine_base("cylinderD_6x8x10")
    zero = np.zeros(base.shape)
    assert np.array_equal(step_split(prepare(base, 0.05), zero, zero), zero)


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_small_config_runs_match_reference(golden, k):
    r = golden.runs
    sysm = pcfg.BUILDERS[k](SMALL[k])
    res = run_simulation(sysm, int(r[f"c{k}_m"]), float(r[f"c{k}_t"]))
    for c in sysm.components:
        assert rel_inf(res.fields[c.name] + c.lift, r[f"c{k}_{c.name}_final"]) <= STEP1_TOL


def test_small_ensemble_members_match_reference(golden):
    from paper_2604_11558_b200.ensemble import run_ensemble

    members = [pcfg.config5_member(i, SMALL[5]) for i in (0, 7, 511)]
    res = run_ensemble(members, 20, 0.02)
    for j, i in enumerate((0, 7, 511)):
        for ci, name in enumerate(("u", "v")):
            assert rel_inf(res.fields[j, ci], golden.runs[f"c5m{i}_{name}_final"]) <= STEP1_TOL
    assert (res.first_bad == INT32_MAX).all()


def _check_samples(full, key, fields, tol):
    """4096 strided samples of the reference's full-size field, and its max-norm."""
    for name, f in fields.items():
        flat = np.asarray(f).ravel()
        idx = full[f"{key}_{name}_idx"]
        ref_max = full[f"{key}_{name}_maxabs"]
        err = np.max(np.abs(flat[idx] - full[f"{key}_{name}_val"])) / ref_max
        assert err <= tol, (key, name, err)
        assert abs(np.max(np.abs(flat)) - ref_max) <= tol * ref_max, (key, name, "max-norm")


_ORACLE_CACHE: dict = {}


def _oracle_physical(key, build, steps, tau):
    """Oracle physical fields after `steps` (cached: both theta modes compare
    against the same CPU run)."""
    hit = _ORACLE_CACHE.get((key, steps))
    if hit is None:
        osys = build()
        hit = orc.physical(osys, orc.integrate(osys, steps, steps * tau))
        _ORACLE_CACHE[(key, steps)] = hit
    return hit


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_full_config_matches_reference_at_steps_1_and_100(golden, k):
    full = golden.full
    sysm = pcfg.BUILDERS[k]()
    m, ts = pcfg.STEPS[k]
    tau = ts / m
    lifts = {c.name: c.lift for c in sysm.components}
    r1 = run_simulation(sysm, 1, tau)
    _check_samples(full, f"f{k}_s1", {n: v + lifts[n] for n, v in r1.fields.items()}, STEP1_TOL)
    r100 = run_simulation(sysm, 100, 100 * tau)
    _check_samples(full, f"f{k}_s100", {n: v + lifts[n] for n, v in r100.fields.items()}, STEP100_TOL)
    # whole fields against the oracle on the same inputs after 1 and 100 steps
    init = [c.initial for c in sysm.components]
    for steps, res, tol in ((1, r1, STEP1_TOL), (100, r100, STEP100_TOL)):
        ref = _oracle_physical(f"config{k}", lambda: ocfg.BUILDERS[k](initial=init), steps, tau)
        for c in sysm.components:
            err = rel_inf(res.fields[c.name] + c.lift, ref[c.name])
            assert err <= tol, (k, steps, c.name, err)


def _ensemble_plan(inputs, tau):
    from paper_2604_11558_b200.ensemble import ensemble_plan

    params = np.stack([[g, 0.1, 0.9] for g in inputs.gammas])
    return ensemble_plan(inputs.template, "schnakenberg", params, tau)


def test_full_ensemble_matches_reference_and_oracle(golden):
    import torch

    full = golden.full
    ens = pcfg.config5_inputs(0, 512)
    plan = _ensemble_plan(ens, 1e-3)
    state = torch.from_numpy(ens.states).cuda()
    bad = torch.full((512, 2), INT32_MAX, dtype=torch.int32, device="cuda")
    plan.run(state, 0, 1, bad)
    s1 = state.cpu().numpy()
    lifts = np.array([1.0, 0.9 / 1.0**2])
    for i in (0, 255, 511):
        _check_samples(full, f"f5m{i}_s1", {"u": s1[i, 0] + lifts[0], "v": s1[i, 1] + lifts[1]}, STEP1_TOL)
    # every member against the oracle after one step
    worst = 0.0
    for i in range(0, 512, 7):
        osys = ocfg.config5_member(i, initial=[ens.states[i, 0], ens.states[i, 1]])
        ref = orc.physical(osys, orc.integrate(osys, 1, 1e-3))
        worst = max(worst, rel_inf(s1[i, 0] + lifts[0], ref["u"]), rel_inf(s1[i, 1] + lifts[1], ref["v"]))
    assert worst <= STEP1_TOL
    plan.run(state, 1, 99, bad)
    s100 = state.cpu().numpy()
    for i in (0, 255, 511):
        _check_samples(full, f"f5m{i}_s100", {"u": s100[i, 0] + lifts[0], "v": s100[i, 1] + lifts[1]},
                       STEP100_TOL)
    # whole fields of 8 members spread over the gamma sweep against the oracle after 100 steps
    for i in (0, 73, 146, 219, 292, 365, 438, 511):
        ref = _oracle_physical(f"member{i}", lambda: ocfg.config5_member(i, initial=[ens.states[i, 0],
                                                                                     ens.states[i, 1]]), 100, 1e-3)
        for c, name in enumerate(("u", "v")):
            err = rel_inf(s100[i, c] + lifts[c], ref[name])
            assert err <= STEP100_TOL, (i, name, err)
    assert (bad.cpu().numpy() == INT32_MAX).all()


@pytest.mark.slow
def test_full_horizon_config1_and_ensemble_members_vs_oracle():
    import torch

    sysm = pcfg.config1()
    res = run_simulation(sysm, 1000, 1.0)
    osys = ocfg.config1(initial=[c.initial for c in sysm.components])
    ref = orc.integrate(osys, 1000, 1.0)
    for c in sysm.components:
        assert rel_inf(res.fields[c.name], ref[c.name]) <= STEP100_TOL
    ens = pcfg.config5_inputs(509, 3)
    plan = _ensemble_plan(ens, 1e-3)
    state = torch.from_numpy(ens.states).cuda()
    bad = torch.full((3, 2), INT32_MAX, dtype=torch.int32, device="cuda")
    plan.run(state, 0, 1000, bad)
    out = state.cpu().numpy()
    osys = ocfg.config5_member(511, initial=[ens.states[2, 0], ens.states[2, 1]])
    ref = orc.physical(osys, orc.integrate(osys, 1000, 1.0))
    assert rel_inf(out[2, 0] + 1.0, ref["u"]) <= STEP100_TOL
    assert rel_inf(out[2, 1] + 0.9, ref["v"]) <= STEP100_TOL


def test_divergence_names_the_oracle_step():
    from paper_2604_11558_b200.models import Kinetics

    sysm = pcfg.config1(SMALL[1])
    wild = type(sysm)(spec=None, components=sysm.components,
                      kinetics=Kinetics("schnakenberg", {"gamma": 3.0e4, "a": 0.1, "b": 0.9}), equilibrium={})
    osys = ocfg.config1(SMALL[1], initial=[c.initial for c in sysm.components])
    osys.params["gamma"] = 3.0e4
    with pytest.raises(orc.OracleDivergence) as ref_err:
        orc.integrate(osys, 200, 0.2)
    with pytest.raises(DivergenceError) as err:
        run_simulation(wild, 200, 0.2, record_every=7)
    assert err.value.step == ref_err.value.step


def test_reruns_are_bitwise_identical():
    sysm = pcfg.config4((10, 12, 10))
    a = run_simulation(sysm, 37, 0.37)
    b = run_simulation(sysm, 37, 0.37)
    for n in a.fields:
        assert np.array_equal(a.fields[n], b.fields[n])


def test_graph_chunks_equal_eager_steps():
    import torch

    sysm = pcfg.config1(SMALL[1])
    geos = [prepare(c.ops, 1e-3) for c in sysm.components]
    plan = SplitPlan(geos, 1, "schnakenberg", sysm.kinetics.param_vector()[None, :])
    init = torch.from_numpy(np.stack([c.initial for c in sysm.components])[None]).cuda()
    bad = torch.full((1, 2), INT32_MAX, dtype=torch.int32, device="cuda")
    a = init.clone()
    plan.run(a, 0, 35, bad)  # two 16-step graph replays + 3 eager steps
    b = init.clone()
    for s in range(35):
        plan.run(b, s, 1, bad)
    assert torch.equal(a, b)


def test_sampling_schedule_and_hook():
    sysm = pcfg.config1(SMALL[1])
    seen = []
    res = run_simulation(sysm, 10, 0.01, record_every=4,
                         diagnostics=lambda st: {n: float(np.mean(v)) for n, v in st.items()},
                         sample_hook=lambda step, t, st: seen.append(step))
    assert seen == [0, 4, 8, 10]
    assert len(res.times) == 4 and len(res.series["u"]) == 4


@pytest.mark.parametrize("kind,params", [
    ("schnakenberg", {"gamma": 100.0, "a": 0.1, "b": 0.9}),
    ("brusselator", {"A": 4.5, "B": 6.96}),
    ("gray_scott", {"F": 0.04, "k": 0.06}),
    ("bvam_eta", {"eta": 0.45, "a": 1.112, "b": -1.01, "h": -1.0, "C": 0.02}),
    ("bvam", {"alpha1": 0.899, "alpha2": 0.2, "alpha3": 0.2, "beta1": -0.91, "beta2": -0.899}),
    ("dib", {"zeta1": 10.0, "zeta2": 10.0, "zeta3": 1.0, "zeta4": 48.0, "zeta5": 0.5, "eta1": 5.0, "eta2": 2.5,
             "eta3": 0.2, "eta5": 1.5}),
])
def test_kinetics_kernel_bitwise_vs_oracle(kind, params):
    import torch

    from paper_2604_11558_b200.models import Kinetics

    base = engine_base("disk_20x36")
    kin = Kinetics(kind, params)
    geos = [prepare(base, 0.01), prepare(base, 0.01)]
    plan = SplitPlan(geos, 2, kind, np.stack([kin.param_vector()] * 2), lifts=[0.25, -0.5])
    rs = np.random.RandomState(3)
    W = rs.randn(2, 2, *base.shape)
    G = torch.empty((2, 2) + base.shape, dtype=torch.float64, device="cuda")
    plan.kinetics_into(torch.from_numpy(W).cuda(), G)
    got = G.cpu().numpy()
    for b in range(2):
        # DIB's r**3: NumPy's SIMD pow is not correctly rounded on AVX-512 hosts
        # (about 3 % of cubes are off by an ulp), so the bitwise reference uses
        # the exactly rounded cube, the value the kernel's cube_rn produces;
        # against NumPy's own pow the kinetics agree to a few ulp
        ref = orc.kinetics(kind, params, {"u": W[b, 0], "v": W[b, 1]}, ["u", "v"], [0.25, -0.5], cube=_exact_cube)
        assert np.array_equal(got[b, 0], ref["u"]), kind
        assert np.array_equal(got[b, 1], ref["v"]), kind
        numpy_ref = orc.kinetics(kind, params, {"u": W[b, 0], "v": W[b, 1]}, ["u", "v"], [0.25, -0.5])
        for c, n in enumerate(("u", "v")):
            assert np.max(np.abs(got[b, c] - numpy_ref[n])) <= 1e-14 * np.max(np.abs(numpy_ref[n])), kind


def _exact_cube(x):
    from fractions import Fraction

    flat = np.asarray(x, dtype=np.float64).ravel()
    return np.array([float(Fraction(float(v)) ** 3) for v in flat]).reshape(np.shape(x))


def test_full_size_ball_reruns_bitwise_identical():
    """Regression guard: partial tiles (n = 100) under the persistent,
    two-CTA-per-SM GEMM once produced run-to-run differences (a clipped bulk
    tensor store; see csrc/gemm.cuh)."""
    import torch

    sysm = pcfg.config4()
    geos = [prepare(c.ops, 1e-2) for c in sysm.components]
    plan = SplitPlan(geos, 1, sysm.kinetics.kind, sysm.kinetics.param_vector()[None, :])
    W = torch.from_numpy(np.stack([c.initial for c in sysm.components])[None]).cuda()
    bad = torch.full((1, 2), INT32_MAX, dtype=torch.int32, device="cuda")
    outs = []
    for _ in range(4):
        s = W.clone()
        plan.run(s, 0, 40, bad)
        outs.append(s.cpu())
    for o in outs[1:]:
        assert torch.equal(outs[0], o)


def test_ball_middle_mode_stage_bitwise_over_many_reruns():
    """Regression guard for the stage-ring release race (a generic-proxy read
    / async-proxy refill WAR, fixed with fence.proxy.async before the empty
    arrive): the n = 100 middle-mode stage, 100 reruns on fixed inputs; the
    unfenced kernel differed in about 1 of 200 reruns."""
    import torch

    sysm = pcfg.config4()
    geos = [prepare(c.ops, 1e-2) for c in sysm.components]
    plan = SplitPlan(geos, 1, sysm.kinetics.kind, sysm.kinetics.param_vector()[None, :], theta="gemm")
    W = torch.from_numpy(np.stack([c.initial for c in sysm.components])[None]).cuda()
    out = torch.empty_like(W)
    for st in plan.step_kernels():
        plan.run_stage(st, W, out)
    first = None
    for _ in range(100):
        plan.run_stage(2, W, out)
        got = plan.workspace(1).clone()
        if first is None:
            first = got
        else:
            assert torch.equal(first, got)


@pytest.mark.parametrize("k,dims", [(1, (5, 7)), (2, (8, 5)), (3, (4, 6, 9)), (4, (5, 6, 7)), (2, (7, 9))])
def test_odd_contiguous_axis_runs_match_oracle(k, dims):
    """Odd last-axis extents (stored padded to even rows inside the plan;
    the caller's arrays stay unpadded): 40 steps, graph chunks included,
    against the oracle on identical inputs."""
    sysm = pcfg.BUILDERS[k](dims)
    m, ts = pcfg.STEPS[k]
    tau = ts / m
    res = run_simulation(sysm, 40, 40 * tau, record_every=17)
    osys = ocfg.BUILDERS[k](dims, initial=[c.initial for c in sysm.components])
    ref = orc.integrate(osys, 40, 40 * tau)
    for c in sysm.components:
        assert rel_inf(res.fields[c.name], ref[c.name]) <= STEP1_TOL, c.name


@pytest.mark.parametrize("cfg", ["2", "7", "8", "9", "11", "12", "13", "18", "19"])
@pytest.mark.parametrize("k,dims", [(2, (24, 16)), (4, (10, 12, 10)), (1, (16, 32)), (3, (8, 16, 16))])
def test_cluster_split_k_gemm_matches_oracle_and_reruns(monkeypatch, cfg, k, dims):
    """Every GEMM stage forced onto one tile configuration: the split-K cluster
    kernels (cfg 7: 2-CTA, cfg 8: 4-CTA clusters, cfg 11: 2-CTA clusters of
    8-warp CTAs, partials reduced over DSMEM in rank order), incl.
    ranks with no k slice at all (K = 16 with 2 or 4 ranks), and the
    non-default single-CTA tiles (cfg 2: 4 warps of 32x32, cfg 9: 8 warps of
    32x16; cfg 18 / 19: the 112-row "tall" tiles of the NN stages, whose warps
    skip their dead 8-row blocks -- TN stages keep their default under these
    two): same results as the oracle within the single-op tolerance and
    bitwise-identical reruns."""
    monkeypatch.setenv("CURVIGPU_TILE_CFG", cfg)
    sysm = pcfg.BUILDERS[k](dims)
    m, t = 6, {1: 6e-3, 2: 6e-3, 3: 3.0, 4: 6e-2}[k]
    a = run_simulation(sysm, m, t)
    b = run_simulation(sysm, m, t)
    osys = ocfg.BUILDERS[k](dims, initial=[c.initial for c in sysm.components])
    ref = orc.physical(osys, orc.integrate(osys, m, t))
    for c in sysm.components:
        assert np.array_equal(a.fields[c.name], b.fields[c.name])
        assert rel_inf(a.fields[c.name] + c.lift, ref[c.name]) <= 1e-12


@pytest.mark.parametrize("variant", [{}, {"CURVIGPU_FRONT_NT256": "1"}, {"CURVIGPU_FRONT_NT64": "1"}])
def test_fused_front_cta_variants_match_oracle_and_each_other(monkeypatch, theta_mode, variant):
    """The fused disk front in each CTA shape (128-thread CTAs at 3/SM, the
    default for large ensembles; 256-thread at 2/SM; 64-thread) on a
    160-run config-5 ensemble (enough items for the 128-thread default; its
    444-CTA grid is not a multiple of the 16 row blocks, so Phi rows are
    reloaded, while the 256- and 64-thread grids reuse them):
    10 steps, members against the oracle, all variants bitwise equal."""
    import torch

    for k, v in variant.items():
        monkeypatch.setenv(k, v)
    monkeypatch.setenv("CURVIGPU_LANES", "1")  # one 160-run plan (two lanes would halve it)
    ens = pcfg.config5_inputs(100, 160)
    plan = _ensemble_plan(ens, 1e-3)
    state = torch.from_numpy(ens.states).cuda()
    bad = torch.full((160, 2), INT32_MAX, dtype=torch.int32, device="cuda")
    plan.run(state, 0, 10, bad)
    out = state.cpu().numpy()
    for j in (0, 77, 159):
        osys = ocfg.config5_member(100 + j, initial=[ens.states[j, 0], ens.states[j, 1]])
        ref = orc.physical(osys, orc.integrate(osys, 10, 1e-2))
        assert rel_inf(out[j, 0] + 1.0, ref["u"]) <= STEP1_TOL
        assert rel_inf(out[j, 1] + 0.9, ref["v"]) <= STEP1_TOL
    key = f"_front_variant_reference_{theta_mode}"  # gemm mode has no fused front: variants agree trivially
    first = globals().get(key)
    if first is None:
        globals()[key] = out
    else:
        assert np.array_equal(out, first)


def test_lanes_give_identical_results(monkeypatch, theta_mode):
    """A plan split into lanes (independent run blocks on their own streams)
    equals the single plan bitwise, including the divergence record; the
    Ensemble's per-lane upload / step / download path equals it too."""
    import torch

    from paper_2604_11558_b200.ensemble import Ensemble

    ens = pcfg.config5_inputs(40, 12, SMALL[5])
    params = np.stack([[g, 0.1, 0.9] for g in ens.gammas])
    params[5, 0] = 5e8  # one member diverges: its first bad step must survive the lane split
    outs = []
    for lanes in (1, 2, 3):
        plan = ensemble_plan_lanes(ens, params, lanes)
        assert plan.lanes == lanes
        state = torch.from_numpy(ens.states).cuda()
        bad = torch.full((12, 2), INT32_MAX, dtype=torch.int32, device="cuda")
        plan.run(state, 0, 30, bad)
        outs.append((state.cpu().numpy(), bad.cpu().numpy()))
        plan.close()
    for o, b in outs[1:]:
        assert np.array_equal(np.nan_to_num(o, nan=7.0), np.nan_to_num(outs[0][0], nan=7.0))
        assert np.array_equal(b, outs[0][1])
    assert (outs[0][1][5] < INT32_MAX).any() and (np.delete(outs[0][1], 5, axis=0) == INT32_MAX).all()
    res = []
    for lanes in ("1", "2"):
        monkeypatch.setenv("CURVIGPU_LANES", lanes)
        e = Ensemble(ens.template, "schnakenberg", params, 1e-3)
        e.load(ens.states)
        out = e.advance(30)
        torch.cuda.synchronize()  # the download is asynchronous (pinned host buffer)
        res.append((out.numpy().copy(), e.first_bad.cpu().numpy()))
    assert np.array_equal(np.nan_to_num(res[0][0], nan=7.0), np.nan_to_num(res[1][0], nan=7.0))
    assert np.array_equal(res[0][1], res[1][1])
    assert np.array_equal(np.nan_to_num(res[0][0], nan=7.0), np.nan_to_num(outs[0][0], nan=7.0))


def ensemble_plan_lanes(inputs, params, lanes):
    from paper_2604_11558_b200.integrators import SplitPlan, prepare

    geos = [prepare(c.ops, 1e-3) for c in inputs.template.components]
    lifts = [float(c.lift) for c in inputs.template.components]
    return SplitPlan(geos, batch=params.shape[0], kinetics="schnakenberg", kin_params=params, lifts=lifts,
                     lanes=lanes)


@pytest.mark.parametrize("dims", [(8, 16, 10), (5, 6, 7), (6, 8, 128), (100, 100, 100)])
def test_ball_chained_polar_products_match_two_stages_bitwise(monkeypatch, theta_mode, dims):
    """The ball's two polar-mode products (x3 V^-1, o Phi_outer, x3 V) run as
    one chained kernel (intermediate in shared memory, zero column blocks
    and k steps skipped; 32- and 16-row tiles) and, under CURVIGPU_NO_CHAIN,
    as two GEMM stages:
    the plans differ by one stage and give bitwise-equal fields after 25
    steps (odd n3 = 7: padded rows; n3 = 128: the chain tile's full width);
    the chained run also matches the oracle."""
    import torch

    sysm = pcfg.BUILDERS[4](dims)
    tau = 1e-2
    geos = [prepare(c.ops, tau) for c in sysm.components]
    kin = sysm.kinetics
    W0 = torch.from_numpy(np.stack([c.initial for c in sysm.components])[None]).cuda()
    outs, nstages = [], []
    for mode in ("14", "15", None):  # chain tile 32 x 128 (default), 16 x 128, two stages
        if mode:
            monkeypatch.delenv("CURVIGPU_NO_CHAIN", raising=False)
            monkeypatch.setenv("CURVIGPU_CHAIN_CFG", mode)
        else:
            monkeypatch.setenv("CURVIGPU_NO_CHAIN", "1")
        plan = SplitPlan(geos, 1, kin.kind, kin.param_vector()[None, :], theta=theta_mode)
        nstages.append(plan.stage_count())
        s = W0.clone()
        bad = torch.full((1, 2), INT32_MAX, dtype=torch.int32, device="cuda")
        plan.run(s, 0, 25, bad)
        outs.append(s.cpu().numpy())
    assert nstages[0] == nstages[1] == nstages[2] - 1
    assert np.array_equal(outs[0], outs[2]) and np.array_equal(outs[1], outs[2])
    if dims != (100, 100, 100):
        osys = ocfg.BUILDERS[4](dims, initial=[c.initial for c in sysm.components])
        ref = orc.integrate(osys, 25, 25 * tau)
        for i, c in enumerate(sysm.components):
            assert rel_inf(outs[0][0, i], ref[c.name]) <= STEP1_TOL, c.name


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [(12, 100, 24), (6, 100, 20), (6, 100, 8)])
def test_ball_with_100_theta_points_and_any_polar_extent_matches_the_oracle(dims):
    """n_theta = 100 takes the 5 x 10 FFT only when the polar extent fills its
    20-line CTAs; other extents must keep the GEMM pair (a 100-point line
    once fell through to the power-of-two Stockham kernel)."""
    from paper_2604_11558_b200.integrators import run_simulation

    got = run_simulation(pcfg.BUILDERS[4](dims), 4, 0.04).fields
    osys = ocfg.BUILDERS[4](dims)
    ref = orc.physical(osys, orc.integrate(osys, 4, 0.04))
    for name in ref:
        assert rel_inf(got[name], ref[name]) <= 1e-12, (dims, name)


@pytest.mark.parametrize("cfg", [None, "19"])
def test_clipped_tma_store_of_partial_tiles_matches_register_path(monkeypatch, theta_mode, cfg):
    """CURVIGPU_TMA_PARTIAL=1 sends partial GEMM tiles through the clipping bulk
    tensor store instead of bounds-checked register stores (re-tested with the
    stage-ring proxy fence in place, profiles/r02_tma_partial.txt): the same
    values bit for bit on a ball with ragged extents, default and tall tiles."""
    if cfg:
        monkeypatch.setenv("CURVIGPU_TILE_CFG", cfg)
    sysm = pcfg.BUILDERS[4]((36, 20, 28))
    a = run_simulation(sysm, 12, 0.12)
    monkeypatch.setenv("CURVIGPU_TMA_PARTIAL", "1")
    b = run_simulation(sysm, 12, 0.12)
    c2 = run_simulation(sysm, 12, 0.12)
    for c in sysm.components:
        assert np.array_equal(a.fields[c.name], b.fields[c.name]), c.name
        assert np.array_equal(b.fields[c.name], c2.fields[c.name]), c.name
