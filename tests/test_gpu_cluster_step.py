"""Small disks advanced by the cluster step kernel (csrc/cluster_disk.cuh: all
steps of cg_run in one kernel, the state in the cluster's shared memory)
against the two-kernel step (CURVIGPU_NO_CLUSTER_STEP=1), the CPU oracle and
the reference's loop semantics (run_simulation, integrators.py:370-430: kinetics
from the common state, guard naming the first bad step, sampling schedule --
tests/test_integrators.py:301-344)."""

import dataclasses

import numpy as np
import pytest

from oracle import configs as ocfg
from oracle import curvi_oracle as orc
from paper_2604_11558_b200 import configs as pcfg
from paper_2604_11558_b200 import models
from paper_2604_11558_b200.ensemble import run_ensemble
from paper_2604_11558_b200.integrators import DivergenceError, run_simulation

from .conftest import rel_inf

pytestmark = pytest.mark.gpu


def _both(monkeypatch, fn):
    monkeypatch.delenv("CURVIGPU_NO_CLUSTER_STEP", raising=False)
    a = fn()
    monkeypatch.setenv("CURVIGPU_NO_CLUSTER_STEP", "1")
    b = fn()
    return a, b


@pytest.mark.parametrize("dims", [(64, 128), (32, 64)])
@pytest.mark.parametrize("m", [1, 2, 17, 100])
def test_cluster_steps_equal_the_two_kernel_step(monkeypatch, dims, m):
    cl, two = _both(monkeypatch, lambda: run_simulation(pcfg.BUILDERS[1](dims), m, m * 1e-3).fields)
    for name in two:
        # phase A is the fused front's arithmetic; the rho product groups k in other 4-blocks
        assert rel_inf(cl[name], two[name]) <= 2e-13 * max(1, m // 10), (dims, m, name)
        assert not np.array_equal(cl[name], pcfg.BUILDERS[1](dims).components[0].initial)


@pytest.mark.parametrize("dims,m,tol", [((64, 128), 1, 1e-10), ((64, 128), 100, 1e-8), ((32, 64), 100, 1e-8),
                                       ((64, 128), 1000, 1e-8)])
def test_cluster_steps_match_the_oracle(dims, m, tol):
    got = run_simulation(pcfg.BUILDERS[1](dims), m, m * 1e-3).fields
    osys = ocfg.BUILDERS[1](dims)
    ref = orc.physical(osys, orc.integrate(osys, m, m * 1e-3))
    for name in ref:
        assert rel_inf(got[name], ref[name]) <= tol, (dims, m, name)


def test_cluster_steps_are_bitwise_reproducible():
    a = run_simulation(pcfg.BUILDERS[1](), 40, 0.04).fields
    b = run_simulation(pcfg.BUILDERS[1](), 40, 0.04).fields
    for name in a:
        assert np.array_equal(a[name], b[name])


def test_sampling_schedule_and_series_equal_the_two_kernel_step(monkeypatch):
    def run():
        system = pcfg.BUILDERS[1]()
        return run_simulation(system, 25, 0.025, record_every=7, diagnostics=models.mean_diagnostics(system))

    cl, two = _both(monkeypatch, run)
    assert np.array_equal(cl.times, two.times) and cl.steps == two.steps
    for key in two.series:
        assert np.allclose(cl.series[key], two.series[key], rtol=1e-13, atol=0)


def test_divergence_names_the_same_first_bad_step(monkeypatch):
    def run():
        system = pcfg.BUILDERS[1]()
        big = [dataclasses.replace(c, initial=c.initial * 40.0) for c in system.components]
        with pytest.raises(DivergenceError) as err:
            run_simulation(dataclasses.replace(system, components=big), 400, 4.0)
        return err.value.step, str(err.value)

    cl, two = _both(monkeypatch, run)
    assert cl == two and cl[0] >= 1


def test_reference_model_on_a_cluster_grid_matches_the_two_kernel_step(monkeypatch):
    """BVAM disk (reference kinetics, models.py:284-290) and the lifted anomalous
    model (models.py:528-532) at 32 x 64 / 64 x 128."""
    for name, dims in (("bvam_disk", {"n_rho": 32, "n_theta": 64}),
                       ("schnakenberg_anomalous_disk", {"n_rho": 64, "n_theta": 128})):
        cl, two = _both(monkeypatch, lambda: run_simulation(models.build_system(name, dims, 3), 30, 0.03).fields)
        for key in two:
            # the anomalous model's fields are lifted (|W| ~ 1e-4 around a lift of 1):
            # rounding at the physical scale is 1e-12 of the lifted one
            assert rel_inf(cl[key], two[key]) <= 1e-11, (name, key)


def test_small_ensembles_run_one_cluster_per_member(monkeypatch):
    """B * NC <= SMs: every member gets its own cluster (shared operators, per-run
    kinetics parameters), and a heterogeneous sweep gets per-run operator sets."""
    members = [pcfg.config5_member(i, (64, 128)) for i in (0, 100, 511)]
    cl, two = _both(monkeypatch, lambda: run_ensemble(members, 20, 0.02).fields)
    assert rel_inf(cl, two) <= 1e-13
    assert np.max(np.abs(cl[0] - cl[2])) > 0
    base = pcfg.BUILDERS[1]((32, 64))
    sweep = []
    for fu, fv in [(1.0, 1.0), (1.0, 0.5), (2.0, 1.5)]:
        comps = [dataclasses.replace(c, ops=dataclasses.replace(c.ops, coeff=c.ops.coeff * f))
                 for c, f in zip(base.components, (fu, fv))]
        sweep.append(dataclasses.replace(base, components=comps))
    cl, two = _both(monkeypatch, lambda: run_ensemble(sweep, 12, 0.012).fields)
    assert rel_inf(cl, two) <= 1e-13
    assert np.max(np.abs(cl[0] - cl[2])) > 1e-6
