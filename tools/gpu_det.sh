python -m paper_2604_11558_b200.build > /dev/null
CURVIGPU_MAX_CARVEOUT=1 REPS=300 STAGE=2 CONFIG=4 python tools/det_stage.py 2>&1 | grep "bad reps"
CURVIGPU_MAX_CARVEOUT=1 REPS=24 python tools/det_stress.py
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
