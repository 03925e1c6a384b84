mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "fused_front or lanes or full_ensemble or small_ensemble or full_horizon or small_config or full_config or kinetics" > gpurun_out/front_tests.log 2>&1; echo "front tests rc=$?"; tail -2 gpurun_out/front_tests.log
CONFIGS=5,1 THETAS=fft timeout 300 python tools/kernel_times.py > gpurun_out/kt_front.jsonl 2>&1; cat gpurun_out/kt_front.jsonl
