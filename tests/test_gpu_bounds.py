"""Out-of-bounds write detection of our own (compute-sanitizer is closed on
the GPU pool: profiles/r02_sanitizer_closed.txt).

Plans created with CURVIGPU_REDZONE=1 put a 1 MiB guard band of a fixed
byte pattern on both sides of every workspace (X, Y, the second state
buffer, the padded-storage copy); the caller's state tensor gets the same
bands here.  Every kernel family runs on shapes with partial tiles, odd
contiguous extents, n = 100, split-K clusters, the chained polar-mode
kernel, the fused front variants and lanes; afterwards no guard byte may
have changed.  Each case also reruns and must be bitwise reproducible.
"""

import os

import numpy as np
import pytest

from paper_2604_11558_b200 import configs as pcfg
from paper_2604_11558_b200.integrators import INT32_MAX, SplitPlan, prepare

pytestmark = pytest.mark.gpu

PAD = 1 << 17  # doubles of guard band around the caller's state (1 MiB)
PATTERN = -1.2345e300


def _guarded(host):
    import torch

    n = host.size
    big = torch.full((n + 2 * PAD,), PATTERN, dtype=torch.float64, device="cuda")
    big[PAD:PAD + n] = torch.from_numpy(np.ascontiguousarray(host).ravel()).cuda()
    return big, big[PAD:PAD + n].view(host.shape)


def _bands_intact(big):
    import torch

    return bool(torch.all(big[:PAD] == PATTERN).item() and torch.all(big[-PAD:] == PATTERN).item())


def _run_case(plan, host, steps):
    import torch

    big, state = _guarded(host)
    bad = torch.full(state.shape[:2], INT32_MAX, dtype=torch.int32, device="cuda")
    plan.run(state, 0, steps, bad)
    torch.cuda.synchronize()
    assert _bands_intact(big), "write past the caller's state"
    assert plan.check_redzones() == 0, "write past a plan workspace"
    return state.cpu().numpy()


CASES = [
    (1, (16, 32), {}), (1, (5, 7), {}), (2, (24, 16), {}), (2, (7, 9), {}), (3, (8, 16, 16), {}),
    (3, (4, 6, 9), {}), (4, (10, 12, 10), {}), (4, (5, 6, 7), {}), (4, (6, 8, 128), {}),
    (4, (100, 100, 100), {}), (4, (10, 12, 10), {"CURVIGPU_NO_CHAIN": "1"}),
    (4, (10, 12, 10), {"CURVIGPU_CHAIN_CFG": "15"}),
] + [(k, d, {"CURVIGPU_TILE_CFG": c}) for c in ("2", "7", "8", "9", "11", "12", "13", "18", "19")
     for k, d in ((2, (24, 16)), (4, (10, 12, 10)))]


@pytest.mark.parametrize("theta", ["gemm", "fft"])
@pytest.mark.parametrize("k,dims,env", CASES, ids=[f"c{k}-{'x'.join(map(str, d))}-{'-'.join(e.values()) or 'default'}"
                                                  for k, d, e in CASES])
def test_no_out_of_bounds_writes(monkeypatch, theta, k, dims, env):
    monkeypatch.setenv("CURVIGPU_REDZONE", "1")
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    sysm = pcfg.BUILDERS[k](dims)
    m, ts = pcfg.STEPS[k]
    geos = [prepare(c.ops, ts / m) for c in sysm.components]
    plan = SplitPlan(geos, 1, sysm.kinetics.kind, sysm.kinetics.param_vector()[None, :], theta=theta)
    host = np.stack([c.initial for c in sysm.components])[None]
    a = _run_case(plan, host, 21)
    b = _run_case(plan, host, 21)
    assert np.array_equal(a, b)
    plan.close()


@pytest.mark.parametrize("variant", [{}, {"CURVIGPU_FRONT_NT256": "1"}, {"CURVIGPU_FRONT_NT64": "1"},
                                     {"CURVIGPU_LANES": "2"}])
def test_ensemble_front_no_out_of_bounds_writes(monkeypatch, variant):
    from paper_2604_11558_b200.ensemble import ensemble_plan

    monkeypatch.setenv("CURVIGPU_REDZONE", "1")
    monkeypatch.setenv("CURVIGPU_LANES", "1")
    for key, val in variant.items():
        monkeypatch.setenv(key, val)
    ens = pcfg.config5_inputs(100, 72, (128, 256))
    params = np.stack([[g, 0.1, 0.9] for g in ens.gammas])
    plan = ensemble_plan(ens.template, "schnakenberg", params, 1e-3, theta="fft")
    a = _run_case(plan, ens.states, 5)
    b = _run_case(plan, ens.states, 5)
    assert np.array_equal(a, b)
    plan.close()
