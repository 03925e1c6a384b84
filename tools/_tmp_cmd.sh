cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_resident.py -x -q -p no:cacheprovider 2>&1 | tail -3
for env in CURVIGPU_RESIDENT=auto; do echo "== $env"; env $env CONFIGS=4 THETAS=fft timeout 600 python tools/kernel_times.py 2>&1; done
timeout 300 python tools/step_times.py 2>&1 | tail -1
