"""GPU parity of the bulk-surface coupled models through
libcurvigpu's C ABI (cg_coupled_kinetics / cg_coupled_run) against the
reference's golden fixtures (tests/golden/make_golden.py make_bulk_surface)
and the CPU oracle (oracle/curvi_oracle.py coupled_kinetics).

Tolerances as in test_gpu_parity: <= 1e-10 relative inf-norm after one step
and after the 20-step small runs, <= 1e-8 after 100 steps; the reaction terms
themselves <= 1e-14 (the NumPy expression order is kept; r**3 goes through
libm pow in NumPy).
"""

import numpy as np
import pytest

from oracle import configs as ocfg
from oracle import curvi_oracle as orc
from paper_2604_11558_b200 import models
from paper_2604_11558_b200.coupled import CoupledPlan
from paper_2604_11558_b200.integrators import INT32_MAX, DivergenceError, SplitPlan, prepare, run_simulation

from .conftest import rel_inf

pytestmark = pytest.mark.gpu

BALL = "bulk_surface_schnakenberg_ball"
CYL = "bsdib_cylinder"
SMALL = {
    "ball_s": (BALL, {"n_rho": 6, "n_theta": 8, "n_phi": 6}, 1, None),
    "ball_odd": (BALL, {"n_rho": 5, "n_theta": 10, "n_phi": 7}, 3, None),
    "ball_zero": (BALL, {"n_rho": 4, "n_theta": 6, "n_phi": 4}, 9,
                  {"zeta2": 0.0, "zeta3": 0.0, "eta1": 0.0, "eta2": 0.0}),
    "cyl_s": (CYL, {"n_rho": 6, "n_theta": 8, "n_z": 5}, 1, None),
    "cyl_odd": (CYL, {"n_rho": 7, "n_theta": 12, "n_z": 4}, 4, None),
}
NAMES = ("u", "v", "r", "s")


@pytest.fixture(autouse=True, params=["gemm", "fft"])
def theta_mode(request, monkeypatch):
    from paper_2604_11558_b200 import integrators

    monkeypatch.setattr(integrators, "THETA_MODE", request.param)
    return request.param


def _system(key):
    name, dims, seed, over = SMALL[key]
    return models.build_system(models.model_spec(name, over), dims, seed)


def _plan(sysm, tau):
    comps = sysm.components
    plan = CoupledPlan([prepare(c.ops, tau) for c in comps], sysm.kinetics, lifts=[c.lift for c in comps])
    plan.load([c.initial for c in comps])
    return plan


@pytest.mark.parametrize("key", sorted(SMALL))
def test_coupled_kinetics_match_reference(golden, key):
    sysm = _system(key)
    plan = _plan(sysm, 1e-3)
    Gb, Gs = plan.kinetics()
    got = [Gb[0, 0], Gb[0, 1], Gs[0, 0], Gs[0, 1]]
    for n, g in zip(NAMES, got):
        assert rel_inf(g.cpu().numpy(), golden.bs[f"{key}_{n}_g0"]) <= 1e-14, n
    plan.close()


@pytest.mark.parametrize("key", sorted(SMALL))
def test_small_coupled_runs_match_reference(golden, key):
    sysm = _system(key)
    m, t = int(golden.bs[f"{key}_m"]), float(golden.bs[f"{key}_t"])
    res = run_simulation(sysm, m, t)
    for n in NAMES:
        assert rel_inf(res.fields[n], golden.bs[f"{key}_{n}_final"]) <= 1e-10, n


def test_zeroed_coupling_reproduces_standalone_bulk_bitwise():
    """tests/test_models.py:272-298 on the GPU: with the exchange switched
    off the coupled run's bulk equals the plain two-component ball run with
    fused Schnakenberg kinetics, bit for bit."""
    import torch

    sysm = _system("ball_zero")
    m, t = 20, 0.002
    res = run_simulation(sysm, m, t, as_torch=True)
    p = sysm.spec.params
    geos = [prepare(c.ops, t / m) for c in sysm.components[:2]]
    plan = SplitPlan(geos, 1, "schnakenberg", np.array([[p["alpha1"], p["alpha2"], p["beta1"]]]))
    state = torch.from_numpy(np.stack([c.initial for c in sysm.components[:2]])[None]).cuda()
    bad = torch.full((1, 2), INT32_MAX, dtype=torch.int32, device="cuda")
    plan.run(state, 0, m, bad)
    assert torch.equal(res.fields["u"], state[0, 0])
    assert torch.equal(res.fields["v"], state[0, 1])


def _check_samples(full, key, fields, tol):
    for name, f in fields.items():
        flat = np.asarray(f).ravel()
        idx = full[f"{key}_{name}_idx"]
        err = np.max(np.abs(flat[idx] - full[f"{key}_{name}_val"])) / full[f"{key}_{name}_maxabs"]
        assert err <= tol, (key, name, err)


@pytest.mark.parametrize("key,name,dims,tau", [
    ("ball_full", BALL, {"n_rho": 30, "n_theta": 50, "n_phi": 30}, 1e-4),
    ("cyl_full", CYL, {"n_rho": 160, "n_theta": 160, "n_z": 20}, 6.25e-3),
])
def test_full_size_models_match_reference_at_steps_1_and_100(golden, key, name, dims, tau):
    """The paper's full-size runs (pkg/configs/ball_full.cfg,
    cylinder_full.cfg): seeded ICs identical, fields after 1 and 100 steps."""
    bs = golden.bs
    sysm = models.build_system(name, dims, 1)
    for c in sysm.components:
        assert np.sum(c.initial) == bs[f"{key}_{c.name}_init_sum"]
    lifts = {c.name: c.lift for c in sysm.components}
    r1 = run_simulation(sysm, 1, tau)
    _check_samples(bs, f"{key}_s1", {n: v + lifts[n] for n, v in r1.fields.items()}, 1e-10)
    r100 = run_simulation(sysm, 100, 100 * tau)
    _check_samples(bs, f"{key}_s100", {n: v + lifts[n] for n, v in r100.fields.items()}, 1e-8)


def test_full_size_ball_whole_field_vs_oracle_after_one_step():
    dims = {"n_rho": 30, "n_theta": 50, "n_phi": 30}
    sysm = models.build_system(BALL, dims, 1)
    r1 = run_simulation(sysm, 1, 1e-4)
    osys = ocfg.bs_ball((30, 50, 30), initial=[c.initial for c in sysm.components])
    ref = orc.integrate(osys, 1, 1e-4)
    for n in NAMES:
        assert rel_inf(r1.fields[n], ref[n]) <= 1e-10, n


@pytest.mark.parametrize("name,dims,m,t", [
    (BALL, {"n_rho": 16, "n_theta": 24, "n_phi": 16}, 100, 100 * 20.0 / 120000),
    (CYL, {"n_rho": 48, "n_theta": 48, "n_z": 12}, 100, 100 * 300.0 / 24000),
])
def test_equilibrium_start_drift(name, dims, m, t):
    """tests/test_acceptance.py:349-380 (criterion 9d): started at the
    equilibrium, the coupled run drifts by <= 1e-12 per step."""
    sysm = models.build_system(name, dims, 1)
    eq = sysm.equilibrium
    flat = type(sysm)(spec=sysm.spec, kinetics=sysm.kinetics, equilibrium=eq, components=[
        type(c)(c.name, c.ops, np.full(c.initial.shape, eq[c.name] - c.lift), c.lift, c.perturbation)
        for c in sysm.components])
    res = run_simulation(flat, m, t)
    drift = max(np.max(np.abs(res.fields[c.name] - (eq[c.name] - c.lift))) for c in flat.components) / m
    assert drift <= 1e-12


def test_divergence_names_the_oracle_step():
    key = "ball_s"
    sysm = _system(key)
    osys = ocfg.bs_ball((6, 8, 6), initial=[c.initial for c in sysm.components])
    with pytest.raises(orc.OracleDivergence) as ref_err:
        orc.integrate(osys, 60, 60 * 0.05)
    with pytest.raises(DivergenceError) as err:
        run_simulation(sysm, 60, 60 * 0.05, record_every=7)
    assert err.value.step == ref_err.value.step
    assert f"'{str(ref_err.value).split()[0]}'" in str(err.value)


def test_graph_chunks_equal_eager_steps():
    import torch

    sysm = _system("cyl_s")
    a = _plan(sysm, 6.25e-3)
    a.run(0, 35)  # two 16-step graph replays + 3 eager steps
    b = _plan(sysm, 6.25e-3)
    for s in range(35):
        b.run(s, 1)
    for x, y in zip(a.fields(), b.fields()):
        assert torch.equal(x, y)
    assert (a.first_bad.cpu().numpy() == INT32_MAX).all()


def test_sampling_schedule_and_hook():
    sysm = _system("ball_s")
    seen = []
    res = run_simulation(sysm, 10, 1e-3, record_every=4,
                         diagnostics=lambda st: {n: float(np.mean(st[n])) for n in NAMES},
                         sample_hook=lambda step, t, st: seen.append(step))
    assert seen == [0, 4, 8, 10]
    assert len(res.series["r"]) == 4
    assert np.allclose(res.times, [0.0, 4e-4, 8e-4, 1e-3])
