mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_front or lanes or full_ensemble or small_ensemble or full_horizon" > gpurun_out/front_tests.log 2>&1; echo "front tests rc=$?"; tail -2 gpurun_out/front_tests.log
for v in pg smem; do
  if [ $v = smem ]; then export CURVIGPU_FRONT_PHI_SMEM=1; fi
  CONFIGS=5 THETAS=fft timeout 200 python tools/kernel_times.py > gpurun_out/kt_front_$v.jsonl 2>&1; echo front $v; tail -1 gpurun_out/kt_front_$v.jsonl
done
