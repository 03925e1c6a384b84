"""The engine's host-side setup (operators, phi1 tables, seeded ICs) against
the reference fixtures.  CPU only; the RNG runs in libcurvigpu.so's host code."""

import numpy as np
import pytest

from paper_2604_11558_b200 import configs as pcfg
from paper_2604_11558_b200 import models, operators as op
from paper_2604_11558_b200.integrators import prepare
from paper_2604_11558_b200.phifun import phi1, phi1_matrix, phi1_outer

from ._cases import CASES, engine_base, oracle_comp
from .conftest import rel_inf


def _rows(o):
    return np.stack([o.a, np.append(o.b, 0), np.append(o.c, 0), o.grid])


def test_rng_bit_exact(golden):
    for seed, rec in golden.rng.items():
        r = models.Xoshiro256pp(int(seed))
        assert [r.next_uint64() for _ in range(16)] == [int(x) for x in rec["raw"]]
        assert np.array_equal(models.Uniform(-1e-3, 1e-3).draw(models.Xoshiro256pp(int(seed)), 17), rec["uniform"])
        assert np.array_equal(models.Normal(1e-5).draw(models.Xoshiro256pp(int(seed)), 17), rec["normal"])


def test_rng_moments():
    z = models.Xoshiro256pp(11).normal(200_000)
    assert abs(z.mean()) < 1e-2 and abs(z.std() - 1.0) < 1e-2
    u = models.Xoshiro256pp(7).uniform(20_000)
    assert u.min() >= 0.0 and u.max() < 1.0


def test_operators_bitwise(golden):
    s = golden.setup
    for n in (2, 3, 10, 64, 100, 256):
        assert op.solve_sigma(n) == s[f"sigma_{n}"]
        assert np.array_equal(_rows(op.build_phi_op(n)[0]), s[f"phi_{n}"])
    for d, n in ((2, 2), (2, 64), (3, 3), (3, 100), (2, 128)):
        assert np.array_equal(_rows(op.build_rho(d, n, 1.0)), s[f"rho{d}_{n}"])
    for n, lam in ((128, -1.95), (16, -1.0), (8, 0.0)):
        assert np.array_equal(_rows(op.build_lambda(n, 1.0, lam)), s[f"lambda_{n}_{lam}"])
    for n in (3, 4, 5, 8, 16):
        fac = op.eig_theta(op.build_theta(n))
        assert np.array_equal(fac.Q, s[f"eigtheta_{n}_Q"])
        assert np.array_equal(fac.lambdas, s[f"eigtheta_{n}_lam"])


def test_eig_and_phi1_bitwise(golden):
    s = golden.setup
    ops = {"rho2_64": op.build_rho(2, 64, 1.0), "phi_100": op.build_phi_op(100)[0],
           "lambda_128": op.build_lambda(128, 1.0, -1.95), "z_16": op.build_z(16, 2.0)}
    for name, o in ops.items():
        fac = op.eig_tridiag(o)
        assert np.array_equal(fac.lambdas, s[f"eig_{name}_lam"])
        assert np.array_equal(np.abs(fac.V), s[f"eig_{name}_Vabs"])
        assert np.array_equal(phi1_matrix(0.0123, fac), s[f"phi1m_{name}"])
    assert np.array_equal(phi1(s["phi1_x"]), s["phi1_y"])
    assert phi1(0.0) == 1.0
    f = s["outer_f"]
    assert np.array_equal(phi1_outer(0.37, [f[:5], f[5:11]]).field, s["outer2"])
    assert np.array_equal(phi1_outer(0.37, [f[:5], f[5:11], f[11:]]).field, s["outer3"])


@pytest.mark.parametrize("name", CASES)
def test_prepare_matches_oracle_operands(name):
    from oracle import curvi_oracle as orc

    g = prepare(engine_base(name), 0.037)
    o = orc.operands(oracle_comp(name), 0.037)
    assert np.array_equal(g.Q_theta, o["Q_theta"])
    if g.phi1_rho is not None:
        assert np.array_equal(g.phi1_rho, o["phi1_rho"])
        assert np.array_equal(g.d_rho, o["d_rho"])
    if g.phi1_phi is not None:
        assert np.array_equal(g.phi1_phi, o["phi1_phi"])
    if g.phi1_z is not None:
        assert np.array_equal(g.phi1_z, o["phi1_z"])
    if g.phi_fac is not None:
        assert np.array_equal(g.phi_fac.V, o["V_phi"])
        assert np.array_equal(g.phi_fac.V_inv, o["Vinv_phi"])
        assert np.array_equal(g.d_phi, o["d_phi"])
    assert np.array_equal(g.phi_mix.field, o["Phi"])
    if g.phi_mix_outer is not None:
        assert np.array_equal(g.phi_mix_outer.field, o["Phi_outer"])


def test_z_neumann_annihilates_constants():
    z = op.build_z_neumann(128, 2.0)
    assert np.max(np.abs(z.toarray().sum(axis=1))) <= 1e-12 * abs(z.a[0])


SMALL = {1: (16, 32), 2: (24, 16), 3: (8, 16, 16), 4: (10, 12, 10), 5: (16, 32)}


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_config_initial_states_bitwise(golden, k):
    sysm = pcfg.BUILDERS[k](SMALL[k])
    for c in sysm.components:
        assert np.array_equal(c.initial, golden.runs[f"c{k}_{c.name}_init"])


@pytest.mark.parametrize("i", [0, 7, 511])
def test_ensemble_member_initial_states_bitwise(golden, i):
    sysm = pcfg.config5_member(i, SMALL[5])
    for c in sysm.components:
        assert np.array_equal(c.initial, golden.runs[f"c5m{i}_{c.name}_init"])
    assert sysm.kinetics.params["gamma"] == 50.0 + 150.0 * i / 511


def test_full_size_initial_states_bitwise(golden):
    full = golden.full
    if not full:
        pytest.skip("full.npz not generated")
    for k in (1, 2, 3, 4):
        sysm = pcfg.BUILDERS[k]()
        for c in sysm.components:
            idx = np.unique(np.linspace(0, c.initial.size - 1, 4096).astype(np.int64))
            assert np.array_equal(c.initial.ravel()[idx], full[f"f{k}_{c.name}_init_sample"])
            assert np.sum(c.initial) == full[f"f{k}_{c.name}_init_sum"]
    ens = pcfg.config5_inputs(0, 512)
    for i in (0, 255, 511):
        for ci, name in enumerate(("u", "v")):
            f = ens.states[i, ci]
            idx = np.unique(np.linspace(0, f.size - 1, 4096).astype(np.int64))
            assert np.array_equal(f.ravel()[idx], full[f"f5m{i}_{name}_init_sample"])


def test_kinetics_descriptor_validation():
    with pytest.raises(NotImplementedError):
        models.Kinetics("mystery", {})
    with pytest.raises(ValueError):
        models.Kinetics("schnakenberg", {"gamma": 1.0})
    k = models.Kinetics("gray_scott", {"F": 0.04, "k": 0.06})
    assert np.array_equal(k.param_vector(), [0.04, 0.06])


@pytest.mark.parametrize("key,name,dims", [
    ("ball_s", "bulk_surface_schnakenberg_ball", {"n_rho": 6, "n_theta": 8, "n_phi": 6}),
    ("cyl_s", "bsdib_cylinder", {"n_rho": 6, "n_theta": 8, "n_z": 5}),
])
def test_bulk_surface_systems_match_reference(golden, key, name, dims):
    """build_system of the bulk-surface models: seeded ICs bitwise, lifts,
    shapes and the coupling descriptor (models.py:570-661)."""
    sysm = models.build_system(name, dims, 1)
    assert [c.name for c in sysm.components] == ["u", "v", "r", "s"]
    for c in sysm.components:
        np.testing.assert_array_equal(c.initial, golden.bs[f"{key}_{c.name}_init"])
    kin = sysm.kinetics
    assert isinstance(kin, models.BulkSurfaceCoupling)
    if kin.kind == "ball":
        assert [c.lift for c in sysm.components] == [0.0] * 4
        assert kin.rho_edge == 1.0 and kin.h > 0
        assert len(kin.param_vector()) == 8
    else:
        assert [c.lift for c in sysm.components] == [1.0, 1.0, 0.0, 0.0]
        assert kin.h == 25.0 / 5
        assert len(kin.param_vector()) == 16
    with pytest.raises(ValueError):
        models.BulkSurfaceCoupling("ball", {"alpha1": 1.0}, h=0.1)
    with pytest.raises(NotImplementedError):
        models.BulkSurfaceCoupling("torus", {}, h=0.1)
