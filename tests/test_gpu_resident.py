"""Resident-operator mode-product kernel (csrc/resident.cuh) against the tiled
TMA-ring kernel (csrc/gemm.cuh), for every epilogue (store, Phi, axpy + guard,
the ball's chained pair) at aligned, ragged (n = 100) and odd extents in both
theta formulations.  Last-mode (TN) products accumulate every output over k in
the tiled kernel's order (sequential 4-blocks), so the chained pair -- the
only stage the default policy hands to the resident kernel -- must agree
BITWISE with the tiled plan; first / middle-mode (NN) products group k as
{4s..4s+3} where the tiled kernel's swizzle-friendly fragments take
{8q + 2t + s}, so forced-resident runs (CURVIGPU_RESIDENT=1) agree to
rounding.  Style of the reference's mode-product tests
(tests/test_tensor.py:40-54)."""

import dataclasses

import numpy as np
import pytest

from oracle import configs as ocfg
from oracle import curvi_oracle as orc
from paper_2604_11558_b200 import configs as pcfg
from paper_2604_11558_b200 import integrators
from paper_2604_11558_b200.integrators import DivergenceError, run_simulation

from .conftest import rel_inf

pytestmark = pytest.mark.gpu

CASES = [
    (1, (16, 32), 4, 0.004), (1, (64, 128), 3, 0.003), (2, (24, 16), 4, 0.004), (2, (64, 128), 3, 0.003),
    (3, (8, 16, 16), 3, 1.5), (3, (64, 128, 128), 2, 1.0), (3, (24, 16, 100), 3, 1.5),
    (4, (10, 12, 10), 3, 0.03), (4, (5, 6, 7), 3, 0.03), (4, (6, 8, 128), 2, 0.02), (4, (40, 20, 64), 3, 0.03),
    (4, (100, 100, 100), 2, 0.02),
]


def _run(monkeypatch, mode, k, dims, m, t):
    monkeypatch.setenv("CURVIGPU_RESIDENT", mode)
    return run_simulation(pcfg.BUILDERS[k](dims), m, t).fields


@pytest.mark.parametrize("theta", ["fft", "gemm"])
@pytest.mark.parametrize("k,dims,m,t", CASES)
def test_forced_resident_runs_equal_the_tiled_kernel_to_rounding(monkeypatch, theta, k, dims, m, t):
    monkeypatch.setattr(integrators, "THETA_MODE", theta)
    tiled = _run(monkeypatch, "0", k, dims, m, t)
    res = _run(monkeypatch, "1", k, dims, m, t)
    for name in tiled:
        assert rel_inf(res[name], tiled[name]) <= 1e-13, (k, dims, theta, name)


@pytest.mark.parametrize("theta", ["fft", "gemm"])
@pytest.mark.parametrize("dims,m,t", [((10, 12, 10), 3, 0.03), ((5, 6, 8), 3, 0.03), ((6, 8, 100), 2, 0.02),
                                      ((40, 20, 64), 3, 0.03), ((100, 100, 100), 2, 0.02)])
def test_resident_chained_pair_equals_the_tiled_chain_bitwise(monkeypatch, theta, dims, m, t):
    """Only the chained polar pair differs between the two plans (the polar
    extent picks the instantiation: 64 and 100-wide, with partial blocks)."""
    monkeypatch.setattr(integrators, "THETA_MODE", theta)
    monkeypatch.setenv("CURVIGPU_RESIDENT_CHAIN_ONLY", "1")
    tiled = _run(monkeypatch, "0", 4, dims, m, t)
    res = _run(monkeypatch, "1", 4, dims, m, t)
    for name in tiled:
        assert np.array_equal(res[name], tiled[name]), (dims, theta, name)


@pytest.mark.parametrize("k,dims,m,t", [(3, (16, 32, 64), 5, 2.5), (4, (20, 16, 100), 5, 0.05), (4, (12, 100, 24), 4, 0.04)])
def test_resident_kernel_runs_match_the_oracle(monkeypatch, k, dims, m, t):
    monkeypatch.setenv("CURVIGPU_RESIDENT", "1")
    got = run_simulation(pcfg.BUILDERS[k](dims), m, t).fields
    osys = ocfg.BUILDERS[k](dims)
    ref = orc.physical(osys, orc.integrate(osys, m, t))
    for name in ref:
        assert rel_inf(got[name], ref[name]) <= 1e-12, (k, name)


def test_default_policy_takes_the_balls_chained_pair(monkeypatch):
    """Full-size ball: the default plan (chained pair resident) equals the
    all-tiled plan bitwise after two steps."""
    monkeypatch.delenv("CURVIGPU_RESIDENT", raising=False)
    auto = run_simulation(pcfg.BUILDERS[4](), 2, 0.02).fields
    tiled = _run(monkeypatch, "0", 4, (100, 100, 100), 2, 0.02)
    for name in tiled:
        assert np.array_equal(auto[name], tiled[name]), name


def test_resident_axpy_epilogue_reports_the_first_diverged_step(monkeypatch):
    """The guard fused into the resident axpy epilogue names the same step as the tiled one."""
    steps = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("CURVIGPU_RESIDENT", mode)
        system = pcfg.BUILDERS[3]((8, 16, 16))
        big = [dataclasses.replace(c, initial=c.initial * 1e11 + 1e11) for c in system.components]
        system = dataclasses.replace(system, components=big)
        with pytest.raises(DivergenceError) as err:
            run_simulation(system, 40, 2000.0)
        steps[mode] = err.value.step
    assert steps["0"] == steps["1"] >= 1
