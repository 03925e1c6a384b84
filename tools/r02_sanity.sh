mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
CONFIGS=4,3,2 THETAS=fft timeout 600 python tools/kernel_times.py > gpurun_out/kernel_times.jsonl 2>&1; echo "kt rc=$?"; cat gpurun_out/kernel_times.jsonl | cut -c1-600
timeout 300 python tools/step_times.py > gpurun_out/step_times.json 2>&1; cat gpurun_out/step_times.json
