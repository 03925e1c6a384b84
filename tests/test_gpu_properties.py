"""Size-independent properties of the split step at BASELINE.json's full grid
sizes, where the oracle would take minutes per case: linearity of one step in
(W, G), theta-rotation equivariance, tau = 0 identity (reference
tests/test_integrators.py:116-123), constants as fixed points
(tests/test_integrators.py:126-142) and independence of an ensemble member from
its position and neighbours in the batch.  All through the C ABI (cg_plan_step
/ cg_run)."""

import numpy as np
import pytest

from paper_2604_11558_b200 import configs as pcfg
from paper_2604_11558_b200 import operators as op
from paper_2604_11558_b200.integrators import ComponentOps, Geometry, prepare, step_split

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["gemm", "fft"])
def theta_mode(request, monkeypatch):
    from paper_2604_11558_b200 import integrators

    monkeypatch.setattr(integrators, "THETA_MODE", request.param)
    return request.param


def _full_base(k):
    """One component's operators on config k's full grid (configs.DIMS)."""
    d = pcfg.DIMS[k]
    if k in (1, 5):
        return ComponentOps(Geometry.DISK, 0.05, rho=op.build_rho(2, d[0], 1.0), theta=op.build_theta(d[1]))
    if k == 2:
        return ComponentOps(Geometry.SPHERE, 0.02, theta=op.build_theta(d[0]), phi=op.build_phi_op(d[1])[0])
    if k == 3:
        return ComponentOps(Geometry.CYLINDER, 0.03, rho=op.build_rho(2, d[0], 1.0), theta=op.build_theta(d[1]),
                            z=op.build_z_neumann(d[2], 2.0))
    return ComponentOps(Geometry.BALL, 0.04, rho=op.build_rho(3, d[0], 1.0), theta=op.build_theta(d[1]),
                        phi=op.build_phi_op(d[2])[0])


def _theta_axis(k):
    return {1: 1, 5: 1, 2: 0, 3: 1, 4: 1}[k]


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_full_size_step_is_linear_in_state_and_forcing(k):
    base = _full_base(k)
    ops = prepare(base, 1e-3)
    rng = np.random.default_rng(100 + k)
    W1, W2, G1, G2 = (rng.standard_normal(base.shape) for _ in range(4))
    a, b = 0.75, -1.5  # exact scalings in binary: only the sums round
    lhs = step_split(ops, a * W1 + b * W2, a * G1 + b * G2)
    rhs = a * step_split(ops, W1, G1) + b * step_split(ops, W2, G2)
    scale = np.max(np.abs(rhs))
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * scale


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_full_size_step_commutes_with_theta_rotation(k, theta_mode):
    base = _full_base(k)
    ops = prepare(base, 1e-3)
    rng = np.random.default_rng(200 + k)
    W, G = rng.standard_normal(base.shape), rng.standard_normal(base.shape)
    ax, shift = _theta_axis(k), 37
    out = step_split(ops, W, G)
    rot = step_split(ops, np.roll(W, shift, axis=ax), np.roll(G, shift, axis=ax))
    # the theta operator is circulant (operators.py build_theta): rotating the
    # input rotates the output; sums regroup, so to rounding, not bitwise
    assert np.max(np.abs(rot - np.roll(out, shift, axis=ax))) <= 1e-12 * np.max(np.abs(out))


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_full_size_zero_tau_is_the_identity_bitwise(k):
    base = _full_base(k)
    rng = np.random.default_rng(300 + k)
    W, G = rng.standard_normal(base.shape), rng.standard_normal(base.shape)
    assert np.array_equal(step_split(prepare(base, 0.0), W, G), W)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_full_size_constants_are_fixed_points(k):
    base = _full_base(k)
    W = np.full(base.shape, -2.25)
    out = step_split(prepare(base, 1e-2), W, np.zeros(base.shape))
    assert np.max(np.abs(out - W)) <= 1e-10


def test_ensemble_members_do_not_depend_on_batch_position_or_neighbours():
    """A config-5 member's fields are a function of its own inputs only: the
    same members in another order, or inside a larger batch, give bitwise the
    same fields (what makes sharding over ranks exact)."""
    from paper_2604_11558_b200.ensemble import run_ensemble

    ids = [3, 500, 41, 7, 260, 128, 99]
    members = {i: pcfg.config5_member(i, pcfg.DIMS[5]) for i in ids + [1, 2, 300, 301, 302]}
    m, t = 12, 0.012
    ref = run_ensemble([members[i] for i in ids], m, t).fields
    perm = [4, 0, 6, 2, 5, 1, 3]
    out = run_ensemble([members[ids[j]] for j in perm], m, t).fields
    for pos, j in enumerate(perm):
        assert np.array_equal(out[pos], ref[j])
    wide_ids = [1, 2] + ids + [300, 301, 302]
    wide = run_ensemble([members[i] for i in wide_ids], m, t).fields
    for j in range(len(ids)):
        assert np.array_equal(wide[2 + j], ref[j])
