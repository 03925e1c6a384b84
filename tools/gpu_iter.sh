# tests + tile sweep + bench (one gpurun call)
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
if [ -n "$SWEEP_CONFIGS" ]; then
python tools/sweep_tiles.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?"; tail -3 gpurun_out/sweep.err
fi
python bench.py --steps 3 --warmup 2 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value', d['value'], 'ms/step', d['ms_per_step'], 'frac_step', d['fp64_frac_of_peak_step'], 'e2e', d['e2e']['value'])
for r in d['kernels']: print(r['kernel'], round(r['achieved'],2), r['unit'], round(r['frac'],3), round(r['ms_per_launch'],4))
for r in d.get('per_config',[]): print(r['config'], 'ms/step', round(r['ms_per_step'],4), 'dofsteps/s %.3e'%r['dof_steps_per_s'], 'gemm_frac', round(r['gemm_chain_frac_fp64_peak'],3))
"
