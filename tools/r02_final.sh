# round-end: full GPU test suite, then the evidence script (bench, reference arm, launch list, ncu summaries, kernel/step times)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
bash tools/gpu_final.sh
