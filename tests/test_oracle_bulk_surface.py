"""Pin the oracle's bulk-surface restatement (oracle/curvi_oracle.py
coupled_kinetics, oracle/configs.py bs_ball / bs_cylinder) against fixtures
produced by the reference's own model_spec/build_system/run_simulation
(tests/golden/make_golden.py make_bulk_surface)."""

import numpy as np
import pytest

from oracle import configs as ocfg
from oracle import curvi_oracle as orc

from .conftest import rel_inf

SMALL = {
    # key: (builder, dims, params)
    "ball_s": ("ball", (6, 8, 6), None),
    "ball_odd": ("ball", (5, 10, 7), None),
    "ball_zero": ("ball", (4, 6, 4), {"zeta2": 0.0, "zeta3": 0.0, "eta1": 0.0, "eta2": 0.0}),
    "cyl_s": ("cyl", (6, 8, 5), None),
    "cyl_odd": ("cyl", (7, 12, 4), None),
}
SEEDS = {"ball_s": 1, "ball_odd": 3, "ball_zero": 9, "cyl_s": 1, "cyl_odd": 4}
NAMES = ("u", "v", "r", "s")


def oracle_system(key, initial=None):
    kind, dims, params = SMALL[key]
    build = ocfg.bs_ball if kind == "ball" else ocfg.bs_cylinder
    return build(dims, seed=SEEDS[key], initial=initial, params=params)


@pytest.mark.parametrize("key", sorted(SMALL))
def test_initial_fields_match_reference(golden, key):
    sysm = oracle_system(key)
    for c in sysm.comps:
        np.testing.assert_array_equal(c.initial, golden.bs[f"{key}_{c.name}_init"])


@pytest.mark.parametrize("key", sorted(SMALL))
def test_coupled_kinetics_match_reference(golden, key):
    init = [golden.bs[f"{key}_{n}_init"] for n in NAMES]
    sysm = oracle_system(key, initial=init)
    g = orc.react(sysm, {n: x.copy() for n, x in zip(NAMES, init)})
    for n in NAMES:
        assert rel_inf(g[n], golden.bs[f"{key}_{n}_g0"]) <= 1e-15, n


@pytest.mark.parametrize("key", sorted(SMALL))
def test_coupled_runs_match_reference(golden, key):
    init = [golden.bs[f"{key}_{n}_init"] for n in NAMES]
    sysm = oracle_system(key, initial=init)
    m, t = int(golden.bs[f"{key}_m"]), float(golden.bs[f"{key}_t"])
    out = orc.integrate(sysm, m, t)
    for n in NAMES:
        assert rel_inf(out[n], golden.bs[f"{key}_{n}_final"]) <= 1e-13, n


def test_zeroed_coupling_reproduces_standalone_bulk():
    """tests/test_models.py:272-298: with zeta2 = zeta3 = eta1 = eta2 = 0 the
    bulk evolves exactly as the uncoupled Schnakenberg ball."""
    key = "ball_zero"
    init = [golden_bs_init(key, n) for n in NAMES]
    sysm = oracle_system(key, initial=init)
    m, t = 20, 0.002
    coupled = orc.integrate(sysm, m, t)
    bulk = orc.System(sysm.comps[:2], "schnakenberg",
                      {"gamma": sysm.params["alpha1"], "a": sysm.params["alpha2"], "b": sysm.params["beta1"]})
    alone = orc.integrate(bulk, m, t)
    np.testing.assert_array_equal(coupled["u"], alone["u"])
    np.testing.assert_array_equal(coupled["v"], alone["v"])


def golden_bs_init(key, name):
    from .conftest import GOLDEN

    return np.load(GOLDEN / "bulk_surface.npz")[f"{key}_{name}_init"]
