"""BASELINE configs 2-4 over their full horizons (configs.STEPS: 2000 / 500 /
1000 steps at full size) in the library's default theta mode against the CPU
oracle on the same initial data -- the reference's end-to-end check
(tests/test_integrators.py:145-165) at the sizes the benchmark runs.
north_star's tolerance after >= 100 steps is 1e-8; measured 1e-13
(profiles/r02_full_horizon.jsonl, tools/full_horizon.py)."""

import numpy as np
import pytest

from oracle import configs as ocfg
from oracle import curvi_oracle as orc
from paper_2604_11558_b200 import configs as pcfg
from paper_2604_11558_b200.integrators import run_simulation

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("k", [2, 3, 4])
def test_full_horizon_matches_oracle(k):
    m, t_star = pcfg.STEPS[k]
    system = pcfg.BUILDERS[k]()
    res = run_simulation(system, m, t_star)
    osys = ocfg.BUILDERS[k](initial=[c.initial for c in system.components])
    ref = orc.physical(osys, orc.integrate(osys, m, t_star))
    for c in system.components:
        got = res.fields[c.name] + c.lift
        err = float(np.max(np.abs(got - ref[c.name])) / np.max(np.abs(ref[c.name])))
        assert err <= 1e-8, (pcfg.NAMES[k], c.name, err)
