python bench.py --steps 3 --warmup 2 --no-extras --theta fft > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json'))
print('value %.4e'%d['value'], 'ms/step', round(d['ms_per_step'],2))
for r in d['kernels']: print('  ', r['kernel'], round(r['achieved'],2), r['unit'], round(r['frac'],3), round(r['ms_per_launch'],4))
"
SWEEP_CONFIGS=1,2,3 SWEEP_CFGS=2 CURVIGPU_THETA=fft python tools/sweep_tiles.py 2>/dev/null | grep '"stage": 0\|"stage": 1' | head
