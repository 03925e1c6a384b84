import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs, integrators
from oracle import configs as ocfg, curvi_oracle as orc
for cfg in ["6", "2"]:
    os.environ["CURVIGPU_TILE_CFG"] = cfg
    sysm = configs.config4()
    tau = 1e-2
    osys = ocfg.config4(initial=[c.initial for c in sysm.components])
    ref1 = orc.integrate(osys, 1, tau)
    for m in (1, 5, 20):
        r = integrators.run_simulation(sysm, m, m * tau)
        refm = orc.integrate(osys, m, m * tau) if m > 1 else ref1
        errs = {n: float(np.max(np.abs(r.fields[n] - refm[n])) / np.max(np.abs(refm[n]))) for n in r.fields}
        print("cfg", cfg, "m", m, errs, flush=True)
        if m == 5:
            d = np.abs(r.fields["v"] - refm["v"])
            idx = np.unravel_index(np.argmax(d), d.shape)
            print("  worst at", idx, d[idx], flush=True)
