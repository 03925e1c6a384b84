python -m paper_2604_11558_b200.build > /dev/null
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python tools/step_times.py
CONFIG=4 THETA=fft REPS=50 python tools/det_stage.py 2>&1 | grep "bad reps"
