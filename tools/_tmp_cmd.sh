cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do CONFIGS=5 THETAS=fft timeout 600 python tools/kernel_times.py 2>&1 | cut -c1-200; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cluster_step.py -x -q -p no:cacheprovider 2>&1 | tail -2
