"""Heterogeneous ensembles (per-run operator sets, cg_desc.ops_per_run):
members that differ in diffusion coefficients run in ONE batched plan, each
against the CPU oracle of its own system, in both theta formulations and
through the disk's fused front (per-run Phi rows and stencil bands)."""

import dataclasses

import numpy as np
import pytest

from oracle import configs as ocfg
from oracle import curvi_oracle as orc
from paper_2604_11558_b200 import configs as pcfg
from paper_2604_11558_b200 import integrators
from paper_2604_11558_b200.ensemble import run_ensemble

from .conftest import rel_inf

pytestmark = pytest.mark.gpu

SMALL = {1: (16, 32), 2: (24, 16), 3: (8, 16, 16), 4: (10, 12, 10), 5: (16, 32)}
STEPS = {1: (12, 0.012), 2: (10, 0.01), 3: (6, 3.0), 4: (8, 0.08), 5: (12, 0.012)}


def _scaled(system, scales):
    comps = [dataclasses.replace(c, ops=dataclasses.replace(c.ops, coeff=c.ops.coeff * f))
             for c, f in zip(system.components, scales)]
    return dataclasses.replace(system, components=comps)


def _oracle(k, dims, system, scales):
    init = [c.initial for c in system.components]
    osys = ocfg.config5_member(3, dims, initial=init) if k == 5 else ocfg.BUILDERS[k](dims, initial=init)
    osys.comps = [dataclasses.replace(c, coeff=c.coeff * f) for c, f in zip(osys.comps, scales)]
    return osys


@pytest.fixture(params=["gemm", "fft"])
def theta_mode(request, monkeypatch):
    monkeypatch.setattr(integrators, "THETA_MODE", request.param)
    return request.param


@pytest.mark.parametrize("k,dims", [(1, SMALL[1]), (2, SMALL[2]), (3, SMALL[3]), (4, SMALL[4]), (5, SMALL[5]),
                                    (5, (32, 64)), (1, (64, 128))])
def test_coefficient_sweep_members_match_their_oracles(theta_mode, k, dims):
    """(5, (32, 64)) and (1, (64, 128)) run the fused disk front (64-thread
    items) with FFT theta: per-run Phi rows and stencil bands."""
    base = pcfg.BUILDERS[k](dims) if k < 5 else pcfg.config5_member(3, dims)
    sweeps = [(1.0, 1.0), (1.0, 0.5), (2.0, 1.5), (0.25, 3.0)]
    members = [_scaled(base, s) for s in sweeps]
    m, t = STEPS[k]
    res = run_ensemble(members, m, t)
    for j, s in enumerate(sweeps):
        osys = _oracle(k, dims, base, s)
        ref = orc.physical(osys, orc.integrate(osys, m, t))
        for ci, c in enumerate(base.components):
            assert rel_inf(res.fields[j, ci], ref[c.name]) <= 1e-12, (k, s, c.name)
    # members really differ (the sweep is not a no-op)
    assert not np.allclose(res.fields[0], res.fields[3])


def test_shared_members_still_use_one_operator_set():
    from paper_2604_11558_b200.ensemble import _check_shared

    members = [pcfg.config5_member(i, SMALL[5]) for i in range(3)]
    assert _check_shared(members)
    assert not _check_shared([members[0], _scaled(members[1], (1.0, 2.0))])
