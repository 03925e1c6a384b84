"""Graph-timed kernels of configs 1-3 under tile configs 2 (64x64), 7 (64x64
split-K over 2-CTA clusters), 8 (4-CTA clusters): each kernel captured 50x in a
CUDA graph and replayed, so launch overhead does not hide small kernels."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2604_11558_b200 import configs
from paper_2604_11558_b200.integrators import INT32_MAX, SplitPlan, prepare


def graph_time(fn, reps=50):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / (5 * reps) * 1e3


def main():
  for k in [int(x) for x in os.environ.get("CONFIGS", "1,2,3").split(",")]:
      for theta in ("fft", "gemm"):
          for cfg in (2, 7, 8):
              os.environ["CURVIGPU_TILE_CFG"] = str(cfg)
              system = configs.BUILDERS[k]()
              m, ts = configs.STEPS[k]
              geos = [prepare(c.ops, ts / m) for c in system.components]
              plan = SplitPlan(geos, 1, system.kinetics.kind, system.kinetics.param_vector()[None, :], theta=theta)
              W = torch.from_numpy(np.stack([c.initial for c in system.components])[None].copy()).cuda()
              out = torch.empty_like(W)
              bad = torch.full((1, 2), INT32_MAX, dtype=torch.int32, device="cuda")
              ks = []
              for st in plan.step_kernels():
                  fl, by = plan.stage_info(st)
                  us = graph_time(lambda: plan.run_stage(st, W, out))
                  ks.append((st, round(us, 2), round(fl / us / 1e6, 2) if fl else None))
              s = W.clone()
              plan.run(s, 0, 32, bad)
              torch.cuda.synchronize()
              e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
              e0.record()
              plan.run(s, 0, 320, bad)
              e1.record()
              e1.synchronize()
              print(json.dumps({"config": k, "theta": theta, "cfg": cfg, "step_us": round(e0.elapsed_time(e1) / 320 * 1e3, 2),
                                "kernels_us_tflops": ks}), flush=True)
              plan.close()


if __name__ == "__main__":
    main()
