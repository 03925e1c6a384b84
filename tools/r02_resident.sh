#!/bin/bash
# resident-operator kernel: parity suites (default policy and forced) + kernel times
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
OUT=gpurun_out/r02_resident.txt
: > $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r02_res_tests_default.log 2>&1
echo "parity default rc=$?" >> $OUT; tail -3 gpurun_out/r02_res_tests_default.log >> $OUT
CURVIGPU_RESIDENT=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hetero_ensemble.py tests/test_gpu_bulk_surface.py -x -q -p no:cacheprovider > gpurun_out/r02_res_tests_forced.log 2>&1
echo "parity forced rc=$?" >> $OUT; tail -3 gpurun_out/r02_res_tests_forced.log >> $OUT
for env in CURVIGPU_RESIDENT=0 CURVIGPU_RESIDENT=auto CURVIGPU_RESIDENT=1; do
  echo "== $env" >> $OUT
  env $env CONFIGS=${CONFIGS:-3,4,5} THETAS=fft,gemm timeout 600 python tools/kernel_times.py >> $OUT 2>&1
done
cat $OUT
