mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
CONFIGS=3,2,1,4 THETAS=fft,gemm timeout 300 python tools/kernel_times.py > gpurun_out/kt_c17.jsonl 2>&1; cut -c1-200 gpurun_out/kt_c17.jsonl
timeout 200 python tools/step_times.py > gpurun_out/st_c17.json 2>&1; tail -1 gpurun_out/st_c17.json
