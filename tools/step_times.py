"""Graph-replayed step time of configs 1-4 (bench.per_config_gpu), both theta modes."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import bench
out = {}
for k in (1, 2, 3, 4):
    for t in ("fft", "gemm"):
        r = bench.per_config_gpu(k, theta=t)
        out[f"c{k}_{t}"] = round(r["ms_per_step"] * 1e3, 2)
print(json.dumps({"pdl": os.environ.get("CURVIGPU_NO_PDL") is None, "us_per_step": out}))
