"""Pin the CPU oracle (oracle/) against fixtures produced by the reference
itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import configs as ocfg
from oracle import curvi_oracle as orc

from ._cases import CASES, oracle_comp
from .conftest import rel_inf


def test_rng_streams_match_reference(golden):
    for seed, rec in golden.rng.items():
        r = orc.Xoshiro(int(seed))
        assert [r.next() for _ in range(16)] == [int(x) for x in rec["raw"]]
        assert np.array_equal(orc.draw(orc.Xoshiro(int(seed)), ("uniform", -1e-3, 1e-3), 17), rec["uniform"])
        assert np.array_equal(orc.draw(orc.Xoshiro(int(seed)), ("normal", 1e-5), 17), rec["normal"])


def test_reference_rng_golden_values():
    # tests/test_models.py:24-31 of the reference
    r = orc.Xoshiro(1)
    assert [r.next() for _ in range(3)] == [14971601782005023387, 13781649495232077965, 1847458086238483744]


def _rows(op):
    return np.stack([op.a, np.append(op.b, 0), np.append(op.c, 0), op.grid])


def test_operator_bands_match_reference(golden):
    s = golden.setup
    for n in (2, 3, 10, 64, 100, 256):
        assert orc.sigma_offset(n) == s[f"sigma_{n}"]
        assert np.array_equal(_rows(orc.polar_stencil(n)), s[f"phi_{n}"])
    for d, n in ((2, 2), (2, 64), (3, 3), (3, 100), (2, 128)):
        assert np.array_equal(_rows(orc.radial_stencil(d, n, 1.0)), s[f"rho{d}_{n}"])
    for n, lam in ((128, -1.95), (16, -1.0), (8, 0.0)):
        assert np.array_equal(_rows(orc.anomalous_stencil(n, 1.0, lam)), s[f"lambda_{n}_{lam}"])


def test_eigen_and_phi1_match_reference(golden):
    s = golden.setup
    for n in (3, 4, 5, 8, 16):
        lam, Q = orc.theta_eigen(orc.theta_stencil(n))
        assert np.array_equal(Q, s[f"eigtheta_{n}_Q"])
        assert np.array_equal(lam, s[f"eigtheta_{n}_lam"])
    ops = {"rho2_64": orc.radial_stencil(2, 64, 1.0), "phi_100": orc.polar_stencil(100),
           "lambda_128": orc.anomalous_stencil(128, 1.0, -1.95), "z_16": orc.axial_stencil_nd(16, 2.0)}
    for name, o in ops.items():
        lam, Q, xi = orc.tridiag_eigen(o)
        assert np.array_equal(lam, s[f"eig_{name}_lam"])
        assert np.array_equal(xi, s[f"eig_{name}_xi"])
        assert np.array_equal(np.abs(xi[:, None] * Q), s[f"eig_{name}_Vabs"])
        assert rel_inf(orc.phi1_dense(0.0123, (lam, Q, xi)), s[f"phi1m_{name}"]) <= 1e-15
    assert np.array_equal(orc.phi1(s["phi1_x"]), s["phi1_y"])
    f = s["outer_f"]
    f1, f2, f3 = f[:5], f[5:11], f[11:]
    assert np.array_equal(orc.phi1_table(0.37, [f1, f2]), s["outer2"])
    assert np.array_equal(orc.phi1_table(0.37, [f1, f2, f3]), s["outer3"])


@pytest.mark.parametrize("name", CASES)
def test_step_matches_reference(golden, name):
    comp = oracle_comp(name)
    for tau in (0.037, 0.0):
        key = f"{name}_tau{tau}"
        W, G = golden.steps[key + "_W"], golden.steps[key + "_G"]
        o = orc.operands(comp, tau)
        assert rel_inf(orc.diffusion(o, W), golden.steps[key + "_MW"]) <= 1e-14
        out = orc.split_step(o, W, G)
        if tau == 0.0:
            assert np.array_equal(out, W)  # tau = 0 is the identity bitwise
        assert rel_inf(out, golden.steps[key + "_out"]) <= 1e-14


SMALL = {1: (16, 32), 2: (24, 16), 3: (8, 16, 16), 4: (10, 12, 10), 5: (16, 32)}


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_config_runs_match_reference(golden, k):
    r = golden.runs
    sysm = ocfg.BUILDERS[k](SMALL[k])  # oracle draws its own IC
    for c in sysm.comps:
        assert np.array_equal(c.initial, r[f"c{k}_{c.name}_init"])
    st = orc.integrate(sysm, int(r[f"c{k}_m"]), float(r[f"c{k}_t"]))
    phys = orc.physical(sysm, st)
    for c in sysm.comps:
        assert rel_inf(phys[c.name], r[f"c{k}_{c.name}_final"]) <= 1e-13


@pytest.mark.parametrize("i", [0, 7, 511])
def test_ensemble_member_runs_match_reference(golden, i):
    r = golden.runs
    sysm = ocfg.config5_member(i, SMALL[5])
    for c in sysm.comps:
        assert np.array_equal(c.initial, r[f"c5m{i}_{c.name}_init"])
    phys = orc.physical(sysm, orc.integrate(sysm, 20, 0.02))
    for c in sysm.comps:
        assert rel_inf(phys[c.name], r[f"c5m{i}_{c.name}_final"]) <= 1e-13


def _check_samples(full, key, phys, tol):
    for name, f in phys.items():
        flat = f.ravel()
        idx = full[f"{key}_{name}_idx"]
        err = np.max(np.abs(flat[idx] - full[f"{key}_{name}_val"])) / full[f"{key}_{name}_maxabs"]
        assert err <= tol, (key, name, err)
        assert abs(np.max(np.abs(flat)) - full[f"{key}_{name}_maxabs"]) <= tol * full[f"{key}_{name}_maxabs"]


@pytest.mark.parametrize("k", [1, 2])
def test_full_size_config_matches_reference_at_step_1_and_100(golden, k):
    full = golden.full
    if not full:
        pytest.skip("full.npz not generated")
    from paper_2604_11558_b200 import configs as pcfg  # host IC generation (C RNG, no GPU)

    sysm_p = pcfg.BUILDERS[k]()
    init = [c.initial for c in sysm_p.components]
    sysm = ocfg.BUILDERS[k](initial=init)
    m, ts = ocfg.CONFIG_STEPS[k]
    tau = ts / m
    _, kept = orc.integrate(sysm, 100, 100 * tau, record={1, 100})
    _check_samples(full, f"f{k}_s1", orc.physical(sysm, kept[1]), 1e-13)
    _check_samples(full, f"f{k}_s100", orc.physical(sysm, kept[100]), 1e-11)
