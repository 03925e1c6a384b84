"""On-device setup: cg_setup_* against the host setup it
replaces (`integrators.prepare`, itself bit-identical to the reference's
prepare -- tests/test_host_setup.py) and against the oracle's operands, in the
style of the reference's operator / phi1 tests
(tests/test_operators.py:281-291 reconstruction and spectrum,
tests/test_phifun.py:38-44 phi1 accuracy, :68-80 phi1_outer)."""

import dataclasses

import numpy as np
import pytest

from oracle import configs as ocfg
from oracle import curvi_oracle as orc
from paper_2604_11558_b200 import configs as pcfg
from paper_2604_11558_b200 import operators as ops
from paper_2604_11558_b200.device_setup import eig_tridiag_device, phi1_device, prepare_device
from paper_2604_11558_b200.ensemble import run_ensemble
from paper_2604_11558_b200.integrators import SplitPlan, prepare, run_simulation
from paper_2604_11558_b200.phifun import phi1

from .conftest import rel_inf

pytestmark = pytest.mark.gpu


def _operators():
    """Every tridiagonal operator family of the reference at BASELINE extents."""
    return {
        "rho_d2_64": ops.build_rho(2, 64, 1.0),
        "rho_d3_100": ops.build_rho(3, 100, 1.0),
        "lambda_128": ops.build_lambda(128, 1.0, -1.95),
        "phi_100": ops.build_phi_op(100)[0],
        "phi_256": ops.build_phi_op(256)[0],
        "z_neumann_128": ops.build_z_neumann(128, 2.0),
        "z_dirichlet_20": ops.build_z(20, 1.5),
        "rho_d2_5": ops.build_rho(2, 5, 0.7),
        "rho_d2_2": ops.build_rho(2, 2, 1.0),
    }


@pytest.mark.parametrize("name", list(_operators()))
def test_device_eigenpairs_reconstruct_the_operator(name):
    op = _operators()[name]
    fac = eig_tridiag_device([op])[0]
    host = ops.eig_tridiag(op)
    scale = np.max(np.abs(host.lambdas))
    # spectrum: ascending, nonpositive, equal to LAPACK's to rounding
    assert np.all(np.diff(fac.lambdas) >= 0)
    assert np.max(fac.lambdas) <= 1e-9 * scale
    assert np.max(np.abs(fac.lambdas - host.lambdas)) <= 1e-13 * scale
    # symmetriser as the host's (libm log/exp on both sides, not bitwise)
    assert rel_inf(fac.xi, host.xi) <= 1e-14
    # orthogonality and reconstruction A = V diag(lambda) V^-1
    n = op.n
    assert np.max(np.abs(fac.Q.T @ fac.Q - np.eye(n))) <= 5e-14
    A = op.toarray()
    assert np.max(np.abs((fac.V * fac.lambdas[None, :]) @ fac.V_inv - A)) <= 1e-12 * np.max(np.abs(A))
    assert np.max(np.abs(fac.V @ fac.V_inv - np.eye(n))) <= 1e-12


def test_batched_eigenpairs_share_distinct_operators():
    a, b = ops.build_rho(2, 64, 1.0), ops.build_rho(2, 64, 0.5)
    facs = eig_tridiag_device([a, b, a])
    assert np.array_equal(facs[0].lambdas, facs[2].lambdas)
    assert np.allclose(facs[1].lambdas, 4.0 * facs[0].lambdas, rtol=1e-12)


def test_nonpositive_offdiagonal_is_rejected_like_the_host():
    op = ops.build_rho(2, 8, 1.0)
    bad = dataclasses.replace(op, b=np.where(np.arange(7) == 3, -1.0, op.b))
    with pytest.raises(ValueError):
        eig_tridiag_device([bad])


def test_phi1_device_matches_host_across_the_branch():
    x = np.concatenate([[0.0, 1e-300, -1e-300, 9.9e-6, -9.9e-6, 1e-5, -1e-5, 1.1e-5],
                        -np.logspace(-9, 4, 400), np.logspace(-9, 1.5, 200)])
    got, want = phi1_device(x), phi1(x)
    small = np.abs(x) < 1e-5
    assert np.array_equal(got[small], want[small])            # Horner branch: same operations
    assert np.max(np.abs(got - want) / np.abs(want)) <= 4e-16  # expm1: 1 ulp libraries on both sides


CASES = [(1, (64, 128)), (2, (512, 256)), (3, (64, 128, 128)), (4, (100, 100, 100)), (5, (128, 256)),
         (1, (5, 8)), (4, (5, 6, 7))]


@pytest.mark.parametrize("k,dims", CASES)
def test_prepare_device_matches_host_prepare(k, dims):
    system = pcfg.BUILDERS[k](dims) if k < 5 else pcfg.config5_member(0, dims)
    m, t = pcfg.STEPS[k]
    tau = t / m
    bases = [c.ops for c in system.components]
    dev = prepare_device(bases, tau)
    for b, g in zip(bases, dev):
        h = prepare(b, tau)
        for name in ("phi1_rho", "phi1_phi", "phi1_z"):
            want = getattr(h, name)
            if want is None:
                assert getattr(g, name) is None
                continue
            assert rel_inf(getattr(g, name), want) <= 1e-12, (k, name)
        assert rel_inf(g.phi_mix.field, h.phi_mix.field) <= 1e-15, k
        if h.phi_mix_outer is not None:
            # phi1(s d_rho lambda_phi): an eigenvalue error of eps * |lambda|_max (either
            # solver's) is amplified by s * max(d_rho) ~ 2e2 at the ball's innermost shell
            assert rel_inf(g.phi_mix_outer.field, h.phi_mix_outer.field) <= 1e-9, k
        for name in ("d_rho", "d_phi", "Q_theta", "lam_theta", "A_rho", "A_theta", "A_phi", "A_z"):
            want = getattr(h, name)
            assert (want is None) == (getattr(g, name) is None)
            if want is not None:
                assert np.array_equal(getattr(g, name), want)
        if h.phi_fac is not None:
            # V, V^-1 enter the ball's polar products as a pair: compare the projector they form
            assert rel_inf(g.phi_fac.V @ g.phi_fac.V_inv, h.phi_fac.V @ h.phi_fac.V_inv) <= 1e-12
            assert np.max(np.abs(g.phi_fac.lambdas - h.phi_fac.lambdas)) <= 1e-13 * np.max(np.abs(h.phi_fac.lambdas))


@pytest.mark.parametrize("k,dims,m,t", [(1, (16, 32), 12, 0.012), (2, (24, 16), 10, 0.01), (3, (8, 16, 16), 6, 3.0),
                                       (4, (10, 12, 10), 8, 0.08), (4, (100, 100, 100), 1, 0.01)])
def test_steps_from_device_operands_match_the_oracle(k, dims, m, t):
    """The whole path on device-prepared operands: north_star's tolerance
    (1e-10 after one step) against the CPU oracle."""
    import torch

    system = pcfg.BUILDERS[k](dims)
    geos = prepare_device([c.ops for c in system.components], t / m)
    plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :])
    state = torch.from_numpy(np.stack([c.initial for c in system.components])[None].copy()).cuda()
    bad = torch.full((1, 2), 2**31 - 1, dtype=torch.int32, device="cuda")
    plan.run(state, 0, m, bad)
    got = state.cpu().numpy()[0]
    osys = ocfg.BUILDERS[k](dims)
    ref = orc.physical(osys, orc.integrate(osys, m, t))
    for ci, c in enumerate(system.components):
        assert rel_inf(got[ci] + c.lift, ref[c.name]) <= 1e-10, (k, c.name)
    plan.close()


def test_heterogeneous_ensemble_with_device_setup_equals_host_setup():
    """A domain-size and coefficient sweep (every member its own eigenproblem):
    device-prepared and host-prepared plans agree to rounding."""
    base = pcfg.config5_member(3, (32, 64))
    members = []
    for j, (fu, fv) in enumerate([(1.0, 1.0), (1.0, 0.5), (2.0, 1.5), (0.25, 3.0), (1.3, 0.7)]):
        comps = []
        for c, f in zip(base.components, (fu, fv)):
            rho = ops.build_lambda(32, 1.0 + 0.1 * j, -1.95)
            o = dataclasses.replace(c.ops, coeff=c.ops.coeff * f, rho=rho,
                                    rho_weights=ops.DiagonalWeights(rho.grid ** -(2.0 - 1.95)))
            comps.append(dataclasses.replace(c, ops=o))
        members.append(dataclasses.replace(base, components=comps))
    host = run_ensemble(members, 12, 0.012, setup="host")
    dev = run_ensemble(members, 12, 0.012, setup="device")
    assert rel_inf(dev.fields, host.fields) <= 1e-11
    assert np.max(np.abs(host.fields[0] - host.fields[4])) > 1e-8  # the sweep is not a no-op


def test_run_simulation_unchanged_by_device_setup_import():
    # the default path still prepares on the host (reference semantics)
    system = pcfg.BUILDERS[1]((16, 32))
    res = run_simulation(system, 3, 0.003)
    assert res.steps == 3
