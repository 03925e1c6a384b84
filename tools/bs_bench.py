import json, sys
sys.path.insert(0, ".")
import bench
for k in bench.BULK_SURFACE:
    print(json.dumps(bench.bulk_surface_gpu(k)), flush=True)
