"""On-device sampling: integral-mean diagnostics evaluated by
cg_weighted_sums inside run_simulation / run_ensemble, and the overlapped
host path for sample_hook, against the reference's own run_simulation
series (tests/golden/diagnostics.npz) and the CPU oracle."""

from pathlib import Path

import numpy as np
import pytest

from oracle import configs as ocfg
from oracle import curvi_oracle as orc
from paper_2604_11558_b200 import configs as pcfg
from paper_2604_11558_b200 import models
from paper_2604_11558_b200.ensemble import run_ensemble
from paper_2604_11558_b200.integrators import DivergenceError, run_simulation

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden" / "diagnostics.npz"
SMALL = {1: (16, 32), 2: (24, 16), 3: (8, 16, 16), 4: (10, 12, 10), 5: (16, 32)}
DIAG_RUNS = {1: (23, 5), 2: (17, 4), 3: (9, 3), 4: (11, 4), 5: (20, 6)}  # (m, record_every), as make_golden
STEPS = {1: (1000, 1.0), 2: (2000, 2.0), 3: (500, 250.0), 4: (1000, 10.0), 5: (1000, 1.0)}
SERIES_TOL = 1e-12  # relative; the device sums in a fixed order, numpy pairwise


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def _system(k):
    return pcfg.BUILDERS[k](SMALL[k]) if k < 5 else pcfg.config5_member(7, SMALL[5])


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_device_mean_series_match_reference(gold, k):
    m, every = DIAG_RUNS[k]
    t = STEPS[k][1] / STEPS[k][0] * m
    sysm = _system(k)
    res = run_simulation(sysm, m, t, record_every=every, diagnostics=models.mean_diagnostics(sysm))
    assert res.times == list(gold[f"c{k}_times"])
    for c in sysm.components:
        ref = gold[f"c{k}_{c.name}_series"]
        got = np.array(res.series[c.name])
        assert got.shape == ref.shape
        assert np.max(np.abs(got - ref)) <= SERIES_TOL * np.max(np.abs(ref))


def test_hook_states_and_host_diagnostics_match_oracle():
    sysm = pcfg.config4(SMALL[4])
    seen = {}
    host_diag = models.mean_diagnostics(sysm)
    res = run_simulation(sysm, 13, 0.13, record_every=5,
                         diagnostics=lambda st: host_diag(st),
                         sample_hook=lambda step, t, st: seen.setdefault(step, (t, st)))
    assert sorted(seen) == [0, 5, 10, 13]
    osys = ocfg.config4(SMALL[4], initial=[c.initial for c in sysm.components])
    _, kept = orc.integrate(osys, 13, 0.13, record={5, 10, 13})
    kept[0] = {c.name: np.asarray(c.initial) for c in sysm.components}
    dev = run_simulation(sysm, 13, 0.13, record_every=5, diagnostics=host_diag)
    for i, step in enumerate([0, 5, 10, 13]):
        t, st = seen[step]
        assert t == step * (0.13 / 13)
        for name, W in st.items():
            ref = kept[step][name]
            assert np.max(np.abs(W - ref)) <= 1e-12 * max(np.max(np.abs(ref)), 1e-300)
            # host-callable and device-evaluated means agree
            assert abs(res.series[name][i] - dev.series[name][i]) <= 1e-14 * max(abs(dev.series[name][i]), 1.0)


def test_hook_not_called_after_divergence():
    from paper_2604_11558_b200.models import Kinetics

    sysm = pcfg.config1(SMALL[1])
    wild = type(sysm)(spec=None, components=sysm.components,
                      kinetics=Kinetics("schnakenberg", {"gamma": 3.0e4, "a": 0.1, "b": 0.9}), equilibrium={})
    seen = []
    with pytest.raises(DivergenceError) as err:
        run_simulation(wild, 200, 0.2, record_every=3, sample_hook=lambda step, t, st: seen.append(step))
    assert seen and max(seen) < err.value.step
    assert seen == list(range(0, max(seen) + 1, 3))


def test_weighted_sums_odd_sizes_deterministic():
    import torch

    rng = np.random.default_rng(5)
    for shape in [(3, 2, 7, 9), (2, 2, 1001), (1, 2, 40000)]:
        W = rng.standard_normal(shape)
        npts = int(np.prod(shape[2:]))
        w = [rng.random(shape[2:]) for _ in range(2)]
        dm = models.DeviceMeans(w, [0.5, -1.0], batch=shape[0])
        Wd = torch.from_numpy(W).cuda()
        a = dm(Wd).cpu().numpy()
        b = dm(Wd).cpu().numpy()
        assert np.array_equal(a, b)
        for bb in range(shape[0]):
            for c in range(2):
                exact = float(np.sum(W[bb, c] * w[c])) + (0.5, -1.0)[c]
                scale = float(np.sum(np.abs(W[bb, c] * w[c]))) + 1.0
                assert abs(a[bb, c] - exact) <= 1e-14 * scale
        assert npts > 0


def test_ensemble_series_equal_single_runs():
    systems = [pcfg.config5_member(i, SMALL[5]) for i in range(4)]
    diag = models.mean_diagnostics(systems[0])
    ens = run_ensemble(systems, 20, 0.02, record_every=6, diagnostics=diag)
    assert ens.series.shape == (4, 2, 5)
    for i, s in enumerate(systems):
        one = run_simulation(s, 20, 0.02, record_every=6, diagnostics=models.mean_diagnostics(s))
        assert ens.times == one.times
        for c, comp in enumerate(s.components):
            np.testing.assert_allclose(ens.series[i, c], one.series[comp.name], rtol=1e-13, atol=0)
