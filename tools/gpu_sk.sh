python -m paper_2604_11558_b200.build > /dev/null
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python tools/step_times.py
CURVIGPU_NO_STREAMK=1 python tools/step_times.py
REPS=100 CONFIG=4 python tools/det_stage.py 2>&1 | grep "bad reps"
timeout 600 python bench.py --steps 3 --warmup 3 --no-extras --theta fft > gpurun_out/bench_fft.json 2> gpurun_out/bench_fft.err
python -c "
import json; d=json.load(open('gpurun_out/bench_fft.json'))
print('fft value %.4e'%d['value'], 'ms/step', round(d['ms_per_step'],2), [(r['kernel'], round(r['ms_per_launch'],4)) for r in d['kernels']])"
