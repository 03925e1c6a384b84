import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.integrators import SplitPlan, prepare
dims = eval(os.environ.get("DIMS", "(100,96,100)"))
n1, n2, n3 = dims
system = configs.config4(dims)
geos = [prepare(c.ops, 1e-2) for c in system.components]
plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :], theta="gemm")
W = torch.from_numpy(np.stack([c.initial for c in system.components])[None]).cuda()
out = torch.empty_like(W)
outs = []
for rep in range(int(os.environ.get("REPS", "16"))):
    for s in plan.step_kernels():
        plan.run_stage(s, W, out)
        if s == 2:
            torch.cuda.synchronize()
            outs.append(plan.workspace(1)[0].cpu().numpy())  # [c, n1, n2, n3]
            break
stack = np.stack(outs)
# majority value per entry
ref = np.median(stack, axis=0)
BM = BN = 64
tiles_m = (n2 + BM - 1) // BM
tiles_n = (n3 + BN - 1) // BN
G = 296
for r, o in enumerate(outs):
    bad = np.argwhere(o != ref)
    if len(bad) == 0:
        continue
    print(f"rep {r}: {len(bad)} bad entries", flush=True)
    c, s, m, n = bad[0]
    f = c  # B = 1
    tile = ((f * n1 + s) * tiles_m + m // BM) * tiles_n + n // BN
    print("  first bad (c, slab, m, n)", (int(c), int(s), int(m), int(n)), "tile", int(tile), "cta", int(tile % G),
          "tile#", int(tile // G), flush=True)
    tiles_hit = set()
    for c, s, m, n in bad:
        tiles_hit.add(((c * n1 + s) * tiles_m + m // BM) * tiles_n + n // BN)
    print("  tiles hit:", sorted(int(t) for t in tiles_hit)[:10], flush=True)
    # compare wrong values with the correct values of the same CTA's other tiles at the same local position
    for cand_off in (-2 * G, -G, G, 2 * G, 1, -1):
        t2 = tile + cand_off
        if t2 < 0 or t2 >= 2 * n1 * tiles_m * tiles_n:
            continue
        tn2 = t2 % tiles_n
        tm2 = (t2 // tiles_n) % tiles_m
        fs = t2 // (tiles_n * tiles_m)
        f2, s2 = fs // n1, fs % n1
        hits = 0
        tot = 0
        for c, s, m, n in bad[:200]:
            ml, nl = m % BM, n % BN
            mm, nn = tm2 * BM + ml, tn2 * BN + nl
            if mm < n2 and nn < n3:
                tot += 1
                hits += int(o[c, s, m, n] == ref[f2, s2, mm, nn])
        print(f"  match vs tile {t2} (offset {cand_off}): {hits}/{tot}", flush=True)
    print("  zeros among bad:", int(np.sum(o[tuple(bad.T)] == 0)), flush=True)
    break
# exhaustive: which tile's correct values match the wrong ones at the same local positions?
for r, o in enumerate(outs):
    bad = np.argwhere(o != ref)
    if len(bad) == 0:
        continue
    ntiles = 2 * n1 * tiles_m * tiles_n
    best = []
    sample = bad[:64]
    for t2 in range(ntiles):
        tn2 = t2 % tiles_n
        tm2 = (t2 // tiles_n) % tiles_m
        fs = t2 // (tiles_n * tiles_m)
        f2, s2 = fs // n1, fs % n1
        hits = 0
        for c, s, m, n in sample:
            mm, nn = tm2 * BM + m % BM, tn2 * BN + n % BN
            if mm < n2 and nn < n3 and o[c, s, m, n] == ref[f2, s2, mm, nn]:
                hits += 1
        if hits > 0:
            best.append((hits, t2))
    best.sort(reverse=True)
    print(f"rep {r}: tiles whose correct values match the wrong ones:", best[:5], flush=True)
    break
