cd "$GRAFT_REPO_ROOT"
CONFIGS=2,3,4 THETAS=fft timeout 600 python tools/kernel_times.py 2>&1 | cut -c1-330
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bulk_surface.py -x -q -p no:cacheprovider 2>&1 | tail -2
