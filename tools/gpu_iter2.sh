python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for v in fused unfused; do
  if [ $v = unfused ]; then export CURVIGPU_NO_FUSED_FRONT=1; fi
  python bench.py --steps 3 --warmup 2 --no-extras > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_$v.json'))
print('$v value %.4e'%d['value'], 'ms/step', round(d['ms_per_step'],2))
for r in d['kernels']: print('  ', r['kernel'], round(r['achieved'],2), r['unit'], round(r['frac'],3), round(r['ms_per_launch'],4))
"
done
