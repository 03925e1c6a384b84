mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
CONFIGS=2,3 THETAS=fft timeout 200 python tools/kernel_times.py > gpurun_out/kt_cta32.jsonl 2>&1; cat gpurun_out/kt_cta32.jsonl
CURVIGPU_NO_CTA32=1 CONFIGS=2,3 THETAS=fft timeout 200 python tools/kernel_times.py > gpurun_out/kt_nocta32.jsonl 2>&1; cat gpurun_out/kt_nocta32.jsonl
timeout 200 python tools/step_times.py > gpurun_out/st_cta32.json 2>&1; tail -1 gpurun_out/st_cta32.json
CURVIGPU_NO_CTA32=1 timeout 200 python tools/step_times.py > gpurun_out/st_nocta32.json 2>&1; tail -1 gpurun_out/st_nocta32.json
