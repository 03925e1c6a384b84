for nb in 2 1; do
  CURVIGPU_FUSED_NBUF=$nb python bench.py --steps 3 --warmup 2 --no-extras --theta fft > gpurun_out/bench_nb$nb.json 2> gpurun_out/bench_nb$nb.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_nb$nb.json'))
print('nbuf $nb value %.4e'%d['value'], 'ms/step', round(d['ms_per_step'],2))
for r in d['kernels']: print('  ', r['kernel'], round(r['achieved'],2), r['unit'], round(r['frac'],3), round(r['ms_per_launch'],4))
"
done
