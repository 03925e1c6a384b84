python -m pytest tests/test_gpu_parity.py -x -q -k "full_config_matches_reference_at_steps_1_and_100" 2>&1 | tail -5
python -m pytest tests/test_gpu_parity.py -x -q -k "full_config_matches_reference_at_steps_1_and_100 and gemm-4" 2>&1 | tail -5
python - <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs, integrators
from oracle import configs as ocfg, curvi_oracle as orc
sysm = configs.config4()
osys = ocfg.config4(initial=[c.initial for c in sysm.components])
ref = orc.integrate(osys, 100, 1.0)
for rep in range(3):
    r = integrators.run_simulation(sysm, 100, 1.0)
    print(rep, {n: float(np.max(np.abs(r.fields[n] - ref[n])) / np.max(np.abs(ref[n]))) for n in r.fields}, flush=True)
PY
