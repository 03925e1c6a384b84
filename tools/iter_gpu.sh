# iteration check: build, GPU parity tests, per-kernel times (configs 5,1-4), config-5 bench line
mkdir -p gpurun_out
python -m paper_2604_11558_b200.build > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
CONFIGS=${CONFIGS:-5,1,2,3,4} THETAS=fft timeout 600 python tools/kernel_times.py > gpurun_out/kernel_times.jsonl 2>&1; echo "kt rc=$?"; cat gpurun_out/kernel_times.jsonl | cut -c1-600
timeout 600 python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('value %.4g ms/step %.4f e2e %.4g' % (d['value'], d['ms_per_step']/1000, d['e2e']['value'])); [print(k['kernel'], round(k['ms_per_launch'],4), round(k['frac'],3)) for k in d['kernels']]"
timeout 300 python tools/step_times.py > gpurun_out/step_times.json 2>&1; cat gpurun_out/step_times.json
